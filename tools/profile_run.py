"""One device-resident MLMC pass of a bench config (for ncu launch lists / full captures).

    python tools/profile_run.py --config c2 [--levels 4] [--passes 1]
"""

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1611_09784_b200.device_runner import DeviceMlmc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--levels", default="", help="comma list of level indices (1-based) to run; default all")
    ap.add_argument("--passes", type=int, default=1)
    ap.add_argument("--warm", type=int, default=0)
    ap.add_argument("--concurrent", action="store_true", help="all levels at once (run_levels, as bench.py)")
    ap.add_argument("--parent-only", action="store_true",
                    help="only the parent (nu) tier of each selected level: one hx_eval_idos_batch_device call")
    args = ap.parse_args()
    kind, levels, nq, p, erange, _ = bench.CONFIGS[args.config]
    lo, hi = bench.grid_range(kind, erange)
    run = DeviceMlmc(bench.make_model(kind), nq, bench.DELTA, bench.SEED, lo, hi, bench.NPTS)
    sel = [int(x) for x in args.levels.split(",")] if args.levels else list(range(1, len(levels) + 1))
    inputs = [run.prepare(lv, levels[lv - 1][0], levels[lv - 1][1], p, lv > 1) for lv in sel]
    torch.cuda.synchronize()
    for _ in range(args.warm):
        for inp in inputs:
            run.run_level(inp)
    torch.cuda.synchronize()
    if args.parent_only:
        for _ in range(args.passes):
            for inp in inputs:
                uniq = torch.unique(inp.parent, dim=0).contiguous()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                run._solve(inp.n, uniq, run.ctx, run.stream)
                torch.cuda.synchronize()
                print(f"level {inp.level} parent tier nu={inp.n} ({uniq.shape[0]} masks): "
                      f"{1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
        return
    if args.concurrent:
        for _ in range(args.warm):
            run.run_levels(inputs)
        for _ in range(args.passes):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            run.run_levels(inputs)
            torch.cuda.synchronize()
            print(f"all levels concurrently: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
        return
    for _ in range(args.passes):
        for inp in inputs:
            t0 = time.perf_counter()
            run.run_level(inp)
            torch.cuda.synchronize()
            print(f"level {inp.level} nu={inp.n} M={inp.M}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
