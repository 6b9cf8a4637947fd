"""Host-side profile of the e2e path (Engine.run_mlmc on config c2): where the wall time goes.

    python tools/e2e_prof.py [--reps 3]
"""
import argparse
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1611_09784_b200 as hx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--rng", default="device", choices=["device", "host"])
    args = ap.parse_args()
    kind, levels, nq, p, erange, _ = bench.CONFIGS[args.config]
    lo, hi = bench.grid_range(kind, erange)
    model = bench.make_model(kind)
    plan = hx.LevelPlan(ns=tuple(n for n, _ in levels), samples=tuple(m for _, m in levels), nq=nq, p_vac=p,
                        delta=bench.DELTA)

    trace = []
    saved = []
    orig = hx.Engine._solve_group

    def traced(self, n, q, words, task_ids, ctx=None):
        t = time.perf_counter()
        out = orig(self, n, q, words, task_ids, ctx)
        trace.append((n, q, len(words), t, time.perf_counter()))
        saved.append((n, q, words))
        return out

    hx.Engine._solve_group = traced
    phases = []

    def timed(name, fn):
        def wrap(self, *a, **k):
            t = time.perf_counter()
            out = fn(self, *a, **k)
            phases.append((name, t, time.perf_counter()))
            return out
        return wrap

    hx.Engine._place_group = timed("place", hx.Engine._place_group)
    hx.Engine._level_finish = timed("finish", hx.Engine._level_finish)
    hx.Engine._level_batch = timed("draw", hx.Engine._level_batch)

    def one(prof=None):
        eng = hx.Engine(model, nq=nq, delta=bench.DELTA, master_seed=bench.SEED, bz_mode="reduced",
                        energy_points=bench.NPTS, energy_range=(lo + 2 * bench.DELTA, hi - 2 * bench.DELTA), rng=args.rng)
        t0 = time.perf_counter()
        if prof:
            prof.enable()
        eng.run_mlmc(plan)
        torch.cuda.synchronize()
        if prof:
            prof.disable()
        return time.perf_counter() - t0

    one()
    all_dt = []
    for _ in range(args.reps):
        trace.clear()
        phases.clear()
        t0 = time.perf_counter()
        dt = one()
        all_dt.append(dt)
        print(f"run_mlmc: {1e3 * dt:.1f} ms", flush=True)
        for name, a, b in sorted(phases, key=lambda x: x[1]):
            print(f"   {name:7s} {1e3 * (a - t0):7.2f} -> {1e3 * (b - t0):7.2f} ms", flush=True)
        for n, q, m, a, b in sorted(trace, key=lambda x: x[3]):
            print(f"   tier n={n} q={q} masks={m}: {1e3 * (a - t0):7.1f} -> {1e3 * (b - t0):7.1f} ms", flush=True)
    import statistics

    print(f"run_mlmc median over {args.reps}: {1e3 * statistics.median(all_dt):.2f} ms, min {1e3 * min(all_dt):.2f} ms")
    # each tier alone (sequential, primary context), same masks as the concurrent run
    from paper_1611_09784_b200.solver import eval_batch
    eng = hx.Engine(model, nq=nq, delta=bench.DELTA, master_seed=bench.SEED, bz_mode="reduced",
                    energy_points=bench.NPTS, energy_range=(lo + 2 * bench.DELTA, hi - 2 * bench.DELTA))
    saved.clear()
    eng.run_mlmc(plan)
    for n, q, words in list(saved):
        for _ in range(2):
            t = time.perf_counter()
            eval_batch(eng.cell(n), eng.kpoints(n, q), words, eng.grid.lo, eng.grid.step, eng.grid.npoints,
                       eng.delta)
            dt = time.perf_counter() - t
        print(f"   tier n={n} q={q} masks={len(words)} alone: {1e3 * dt:7.1f} ms", flush=True)
    pr = cProfile.Profile()
    print(f"profiled run_mlmc: {1e3 * one(pr):.1f} ms")
    pstats.Stats(pr).sort_stats("cumtime").print_stats(30)
    pstats.Stats(pr).sort_stats("tottime").print_stats(20)


if __name__ == "__main__":
    main()
