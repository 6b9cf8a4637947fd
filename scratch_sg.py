import sys, time
import numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle")
import paper_1611_09784_b200 as hx
from paper_1611_09784_b200 import _lib
from paper_1611_09784_b200.sampling import sample_masks
from paper_1611_09784_b200.solver import eval_batch
LO_G, HI_G, NPTS = -6.580201874549387, 14.863393148450246, 201
model = hx.GrapheneNNModel(); spec = model.lattice_spec()
sc = hx.build_supercell(spec, 8); cell = hx.compile_cell(model, sc)
kp = np.ascontiguousarray(hx.make_bz_grid(spec, 8, 4, "reduced").kpoints)
step = (HI_G - LO_G) / (NPTS - 1)
words = sample_masks(sc.nunits, 0.05, 1, 2, 0, 1024)
def run(**o):
    with _lib.options(**o):
        for _ in range(2): eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(5): eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
        torch.cuda.synchronize(); return (time.perf_counter() - t) / 5 * 1e3
for o in ({}, {"HX_SMALL_GRAM": 0}, {}):
    print(o, "%.3f ms" % run(**o), flush=True)
