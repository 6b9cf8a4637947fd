"""Summarise an ncu --csv launch list by kernel name: time (gpu__time_duration.sum) and, when the list
also has it, warp instructions (smsp__inst_executed.sum)."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def summarise(path, top=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [set(), 0.0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        val = float(r[vi].replace(",", ""))
        agg[name][0].add(r[0])
        if r[mi] == "gpu__time_duration.sum":
            agg[name][1] += val * SCALE[r[ui]]
        elif r[mi] == "smsp__inst_executed.sum":
            agg[name][2] += val
    tot = sum(x[1] for x in agg.values())
    out = []
    for k, (ids, ms, inst) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        n = len(ids)
        extra = f"  inst={inst / 1e9:7.3f}G" if inst else ""
        out.append(f"{ms:10.2f} ms {100 * ms / tot:5.1f}%  launches={n:5d}  avg={ms / n:9.4f} ms{extra}  {k}")
    out.append(f"total {tot:.2f} ms")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None))
