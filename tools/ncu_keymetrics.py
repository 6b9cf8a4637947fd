"""Key metrics per kernel from an ncu --set full report (raw page csv on stdin)."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration_ms"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_pipe_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp_inst"),
]
rows = list(csv.reader(sys.stdin))
h, units = rows[0], rows[1]
ki = h.index("Kernel Name")
for r in rows[2:]:
    out = [r[ki].split("(")[0][:48]]
    for k, nm in KEYS:
        if k in h:
            i = h.index(k)
            out.append(f"{nm}={r[i]}{units[i] if units[i] not in ('', '%') else ''}")
    print("  ".join(out))
