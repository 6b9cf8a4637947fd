"""Start / end of every (level, tier) solve of one concurrent device-resident pass, relative to the step start.

    python tools/timeline.py --config c2
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1611_09784_b200.device_runner import DeviceMlmc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--warm", type=int, default=3)
    args = ap.parse_args()
    kind, levels, nq, p, erange, _ = bench.CONFIGS[args.config]
    lo, hi = bench.grid_range(kind, erange)
    run = DeviceMlmc(bench.make_model(kind), nq, bench.DELTA, bench.SEED, lo, hi, bench.NPTS)
    inputs = [run.prepare(lv, levels[lv - 1][0], levels[lv - 1][1], p, lv > 1) for lv in range(1, len(levels) + 1)]
    for _ in range(args.warm):
        run.run_levels(inputs)
    torch.cuda.synchronize()
    run.record = True
    run.records = []
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(run.stream)
    run.run_levels(inputs)
    t1.record(run.stream)
    torch.cuda.synchronize()
    print(f"step {t0.elapsed_time(t1):.2f} ms")
    for r in sorted(run.records, key=lambda r: -r["N"]):
        a, b = r["events"]
        print(f"N={r['N']:5d} masks={r['unique']:5d} nk={r['nk']:3d}  start {t0.elapsed_time(a):7.2f}  end {t0.elapsed_time(b):7.2f}"
              f"  ({a.elapsed_time(b):6.2f} ms)")


if __name__ == "__main__":
    main()
