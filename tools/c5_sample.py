"""One c5 batch of one matrix size (for ncu executed-flop counts per matrix):
    python tools/c5_sample.py --n 512 --batch 200
Same inputs as bench.py's c5 sweep (seeded masks, one generic k-point), a smaller batch."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1611_09784_b200 as hx  # noqa: E402
from paper_1611_09784_b200.sampling import sample_masks  # noqa: E402
from paper_1611_09784_b200.solver import eval_batch  # noqa: E402

SHAPES = {32: (4, 4), 64: (4, 8), 128: (8, 8), 256: (8, 16), 512: (16, 16), 1024: (16, 32), 2048: (32, 32)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, required=True)
    ap.add_argument("--batch", type=int, default=200)
    a = ap.parse_args()
    nu, nu2 = SHAPES[a.n]
    model = hx.GrapheneNNModel()
    sc = hx.build_supercell(model.lattice_spec(), nu, nu2)
    cell = hx.compile_cell(model, sc)
    b1, b2 = model.lattice_spec().reciprocal_vectors()
    kp = np.ascontiguousarray((b1 / (3 * nu) + b2 / (3 * nu2)).reshape(1, 2))
    lo, hi = bench.grid_range("graphene", None)
    words = sample_masks(sc.nunits, 0.05, bench.SEED, 5, 0, a.batch)
    eval_batch(cell, kp, words, lo, (hi - lo) / (bench.NPTS - 1), bench.NPTS, bench.DELTA)
    print(f"n={a.n} batch={a.batch} done")


if __name__ == "__main__":
    main()
