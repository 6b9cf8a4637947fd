"""Executed FP64 work per kernel from an ncu --csv launch list with the metrics
gpu__time_duration.sum, sm__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum and
sm__inst_executed_pipe_tensor_subpipe_dmma.sum (DMMA m8n8k4.f64 = 8*8*4 FMAs = 512 flops per warp
instruction; DFMA = 2 flops, DMUL/DADD = 1)."""
import collections
import csv
import json
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
W = {"sm__sass_thread_inst_executed_op_dfma_pred_on.sum": 2.0, "sm__sass_thread_inst_executed_op_dmul_pred_on.sum": 1.0,
     "sm__sass_thread_inst_executed_op_dadd_pred_on.sum": 1.0, "sm__inst_executed_pipe_tensor_subpipe_dmma.sum": 512.0}


def main(path, top=20, json_out=None, passes=1, label=""):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: {"ms": 0.0, "flops": 0.0, "dmma_flops": 0.0, "ids": set()})
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        a = agg[name]
        a["ids"].add(r[0])
        val = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            a["ms"] += val * SCALE[r[ui]]
        elif r[mi] in W:
            a["flops"] += W[r[mi]] * val
            if "dmma" in r[mi]:
                a["dmma_flops"] += W[r[mi]] * val
    tot_ms = sum(a["ms"] for a in agg.values())
    tot_fl = sum(a["flops"] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"])[:top]:
        tf = a["flops"] / (a["ms"] * 1e-3) / 1e12 if a["ms"] else 0.0
        out.append(f"{a['ms']:9.2f} ms  {a['flops'] / 1e9:9.1f} GFLOP exec ({100 * a['dmma_flops'] / max(a['flops'], 1):5.1f}% DMMA)"
                   f"  {tf:6.2f} TFLOP/s  launches={len(a['ids']):4d}  {k}")
    out.append(f"total {tot_ms:.2f} ms, {tot_fl / 1e9:.1f} GFLOP executed FP64, {tot_fl / (tot_ms * 1e-3) / 1e12:.2f} TFLOP/s "
               "averaged over the serialised kernel time")
    print("\n".join(out))
    res = {"label": label, "source_csv": path, "passes": passes, "serialised_ms_per_pass": tot_ms / passes,
           "executed_gflop_per_pass": tot_fl / 1e9 / passes,
           "dmma_gflop_per_pass": sum(a["dmma_flops"] for a in agg.values()) / 1e9 / passes,
           "kernels": {k: {"ms": a["ms"] / passes, "gflop": a["flops"] / 1e9 / passes, "launches": len(a["ids"])}
                       for k, a in agg.items()}}
    if json_out:
        with open(json_out, "w") as f:
            json.dump(res, f, indent=1)
    return res


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("top", nargs="?", type=int, default=20)
    ap.add_argument("--json", default=None)
    ap.add_argument("--passes", type=int, default=1)
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    main(a.csv, a.top, a.json, a.passes, a.label)
