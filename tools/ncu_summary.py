"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
    tot = sum(x[1] for x in agg.values())
    out = []
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{ms:10.2f} ms {100 * ms / tot:5.1f}%  launches={n:5d}  avg={ms / n:9.4f} ms  {k}")
    out.append(f"total {tot:.2f} ms")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
