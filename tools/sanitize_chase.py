"""Small workloads for compute-sanitizer (racecheck / synccheck / memcheck) over the flag-pipelined bulge-chase
kernels and the stage-1 kernels: every chase variant the bench selects (real chase with 1/4/16 warps per matrix,
the clustered real chase, the complex chase, the Hermitian chase of the table tier) on a couple of matrices.

    compute-sanitizer --tool racecheck python tools/sanitize_chase.py
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_1611_09784_b200 as hx  # noqa: E402
from paper_1611_09784_b200 import _lib  # noqa: E402
from paper_1611_09784_b200.sampling import sample_masks  # noqa: E402
from paper_1611_09784_b200.solver import eval_batch  # noqa: E402

LO, HI, NPTS = -6.580201874549387, 14.863393148450246, 201
CASES = [  # (label, model, nu, q, options)
    ("real chase NW=16", "graphene", 16, 2, {"HX_CHASE_RNW": 16}),
    ("real chase NW=4", "graphene", 16, 2, {"HX_CHASE_RNW": 4}),
    ("real chase NW=1", "graphene", 16, 2, {"HX_CHASE_RNW": 1}),
    ("real chase cluster 2", "graphene", 12, 1, {"HX_CHASE_RCL": 2}),
    ("complex chase", "graphene", 12, 3, {}),
    ("hermitian chase (table)", "table", 6, 1, {}),
]


def main():
    sel = sys.argv[1:]
    for label, kind, nu, q, opts in CASES:
        if sel and not any(s in label for s in sel):
            continue
        model = hx.load_coupling_table(ROOT / "tests/golden/synthetic_11band.tbc") if kind == "table" \
            else hx.GrapheneNNModel()
        sc = hx.build_supercell(model.lattice_spec(), nu)
        cell = hx.compile_cell(model, sc)
        kp = hx.make_bz_grid(model.lattice_spec(), nu, q, "reduced").kpoints[:2]
        words = sample_masks(sc.nunits, 0.05, 7, 1, 0, 2)
        with _lib.options(**opts):
            curves, _, status = eval_batch(cell, kp, words, LO, (HI - LO) / (NPTS - 1), NPTS, 0.01)
        print(f"{label}: status {np.unique(status)}, curve end {curves[0, -1]:.6f}", flush=True)


if __name__ == "__main__":
    main()
