"""Per-launch durations from an ncu --csv launch list, filtered by a kernel-name substring."""
import csv
import sys

S = {"ns": 1e-6, "us": 1e-3, "ms": 1, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1}
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi, ui, gi, bi = (h.index(x) for x in ("Kernel Name", "Metric Value", "Metric Unit", "Grid Size", "Block Size"))
pat = sys.argv[2:] or [""]
mi = h.index("Metric Name") if "Metric Name" in h else None
for r in rows[hi + 1:]:
    if mi is not None and r[mi] != "gpu__time_duration.sum":
        continue
    if any(p in r[ki] for p in pat):
        print(f"{float(r[vi].replace(',', '')) * S[r[ui]]:10.3f} ms  grid={r[gi]:>16} block={r[bi]:>12}  {r[ki].split('(')[0][:50]}")
