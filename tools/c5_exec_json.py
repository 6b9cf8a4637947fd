"""Collect per-size executed FP64 (tools/ncu_flops.py --json outputs of tools/c5_sample.py runs) into
profiles/r02_fp64_executed_c5.json: {"per_matrix_gflop": {n: GFLOP per matrix}}.
    python tools/c5_exec_json.py out.json n1:batch1:file1.json n2:batch2:file2.json ..."""
import json
import sys

out = {"label": "c5 executed FP64 per matrix (ncu counts of one tools/c5_sample.py batch per size)",
       "per_matrix_gflop": {}, "sources": {}}
for arg in sys.argv[2:]:
    n, b, f = arg.split(":", 2)
    d = json.load(open(f))
    out["per_matrix_gflop"][n] = d["executed_gflop_per_pass"] / int(b)
    out["sources"][n] = {"batch": int(b), "executed_gflop": d["executed_gflop_per_pass"],
                         "serialised_ms": d["serialised_ms_per_pass"]}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out["per_matrix_gflop"]))
