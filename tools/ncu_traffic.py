"""DRAM traffic per kernel from an ncu --csv launch list with dram__bytes_read.sum, dram__bytes_write.sum
and gpu__time_duration.sum (one hx_eval_idos_batch_device call of a tier = one "launch" of the roofline)."""
import collections
import csv
import sys

SCALE_T = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
SCALE_B = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1.0}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: {"ms": 0.0, "rd": 0.0, "wr": 0.0, "ids": set()})
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[ki].split("(")[0].strip().startswith(("void hx::", "hx::")):
            continue
        a = agg[r[ki].split("(")[0]]
        a["ids"].add(r[0])
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            a["ms"] += v * SCALE_T[r[ui]]
        elif r[mi] == "dram__bytes_read.sum":
            a["rd"] += v * SCALE_B[r[ui]]
        elif r[mi] == "dram__bytes_write.sum":
            a["wr"] += v * SCALE_B[r[ui]]
    tot = {"ms": 0.0, "rd": 0.0, "wr": 0.0}
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
        gbs = (a["rd"] + a["wr"]) / (a["ms"] * 1e-3) / 1e9 if a["ms"] else 0.0
        print(f"{a['ms']:9.2f} ms  read {a['rd'] / 1e9:8.3f} GB  write {a['wr'] / 1e9:8.3f} GB  {gbs:7.1f} GB/s"
              f"  launches={len(a['ids']):4d}  {k}")
        for x in tot:
            tot[x] += a[x]
    print(f"total (hx kernels) {tot['ms']:.2f} ms, DRAM read {tot['rd'] / 1e9:.3f} GB + write {tot['wr'] / 1e9:.3f} GB "
          f"= {(tot['rd'] + tot['wr']) / 1e9:.3f} GB")
    return tot


if __name__ == "__main__":
    main(sys.argv[1])
