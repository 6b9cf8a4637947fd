"""Benchmark of the hexmc hot path on B200: IDOS samples/s per MLMC level (BASELINE.json metric).

Default workload = BASELINE config 2 (graphene MLMC, nu = 4/8/16/32, nq = 32 -> q = 8/4/2/1,
M = 4096/1024/256/64, p = 0.05, 201 energies, CV quarters on levels 2-4; nq = 24 of the config text is
rejected by the reference itself, SURVEY finding 4).  One step = one full MLMC pass over all levels.

  value : device-resident pipeline (masks already in HBM) -> samples/s over the whole job (all ranks)
  e2e   : the public Engine API (host RNG, host dedup, H2D masks, D2H curves), same metric
  roofline : batched eigensolve of the dominant level tier, algorithmic 16/3 d^3 FP64 flops per
             (sample, k) matrix / its CUDA-event time, against a live cuBLAS ZGEMM FP64 peak
  cpu_baseline : the reference implementation (baseline/_ref, hexmc) on the host cores, bounded sample

`--impl reference` times the reference's own CPU implementation on this box instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

LO_G, HI_G = -6.580201874549387, 14.863393148450246  # reference auto grid for graphene (fx/*/summary.json)
TABLE = ROOT / "tests" / "golden" / "synthetic_11band.tbc"

CONFIGS = {
    # name: (model, levels [(nu, M)], nq, p, energy range or None, description)
    "c1": ("graphene", [(4, 1000)], 24, 0.05, None, "graphene MC nu=4 q=6 M=1000"),
    "c2": ("graphene", [(4, 4096), (8, 1024), (16, 256), (32, 64)], 32, 0.05, None,
           "graphene MLMC nu=4/8/16/32 nq=32 M=4096/1024/256/64"),
    "c3": ("table", [(4, 2048), (8, 512), (16, 128)], 16, 0.05, (-2.932, 4.740),
           "synthetic 11-band table MLMC nu=4/8/16 nq=16 M=2048/512/128"),
}
SEED = 2026
DELTA = 0.01
NPTS = 201


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def make_model(kind):
    import paper_1611_09784_b200 as hx

    return hx.GrapheneNNModel() if kind == "graphene" else hx.load_coupling_table(TABLE)


def grid_range(kind, erange):
    if erange is None:
        return LO_G, HI_G
    return erange[0] - 2 * DELTA, erange[1] + 2 * DELTA


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def fp64_peak_live(dev):
    """cuBLAS complex128 GEMM (4096^3, 8 flops per complex FMA), best of 5 — the FP64 roofline denominator."""
    import torch

    n = 4096
    a = torch.randn(n, n, dtype=torch.complex128, device=dev)
    b = torch.randn(n, n, dtype=torch.complex128, device=dev)
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize(dev)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 8.0 * n**3 / (best * 1e-3) / 1e12


def flush_l2(buf):
    buf.add_(1.0)


# ---------------------------------------------------------------------------------------------------
def reference_engine_run(kind, levels, nq, p, erange, frac, workers):
    """The reference (baseline/_ref hexmc) on a bounded sample: M_l * frac samples per level."""
    ref = ROOT / "baseline" / "_ref"
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_hexmc")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import hexmc  # noqa: F401
    from hexmc.runner import Engine

    model = hexmc.GrapheneNNModel() if kind == "graphene" else hexmc.load_coupling_table(TABLE)
    eng = Engine(model, nq=nq, delta=DELTA, master_seed=SEED, workers=workers, bz_mode="reduced",
                 energy_points=NPTS, energy_range=erange)
    per_level = []
    for lvl, (nu, M) in enumerate(levels, start=1):
        m = max(1, int(round(M * frac)))
        t0 = time.perf_counter()
        s = eng.sample_level(lvl, nu, m, p, with_cv=lvl > 1)
        dt = time.perf_counter() - t0
        per_level.append({"nu": nu, "M": m, "seconds": dt, "cache_hits": s.stats.cache_hits})
    return per_level


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    kind, levels, nq, p, erange, desc = CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    frac = args.ref_fraction
    try:
        # warm-up: one small level (loky spawn + numba load), then timed steps
        for _ in range(max(1, args.warmup)):
            reference_engine_run(kind, levels[:1], nq, p, erange, min(frac, 16 / levels[0][1]), cores)
        step_vals, step_ms, last = [], [], None
        for _ in range(args.steps):
            per = reference_engine_run(kind, levels, nq, p, erange, frac, cores)
            tot_s = sum(x["seconds"] for x in per)
            tot_m = sum(x["M"] for x in per)
            step_vals.append(tot_m / tot_s)
            step_ms.append(tot_s * 1e3)
            last = per
    except Exception as exc:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"reference run failed: {exc!r}"}))
        return 0
    value = statistics.median(step_vals)
    line = {
        "metric": "IDOS samples/sec per MLMC level (graphene MLMC, BASELINE config 2)" if args.config == "c2"
        else f"IDOS samples/sec ({desc})",
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(step_ms), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded reference sampler)", "impl": "reference",
        "config": {"workload": desc, "bz_mode": "reduced", "levels": last, "sample_fraction": frac},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "reference",
                         "sample": f"each step = every level with M_l x {frac} samples, reference Engine "
                                   f"workers={cores} (1 BLAS thread each)"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hx", choices=["hx", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--ref-fraction", type=float, default=1.0 / 16.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_1611_09784_b200 as hx
    from paper_1611_09784_b200 import _lib
    from paper_1611_09784_b200.device_runner import DeviceMlmc, kept_dims

    kind, levels, nq, p, erange, desc = CONFIGS[args.config]
    lo, hi = grid_range(kind, erange)
    model = make_model(kind)
    runner = DeviceMlmc(model, nq, DELTA, SEED, lo, hi, NPTS, device=local)

    def barrier():
        if world > 1:
            dist.barrier()

    inputs = [runner.prepare(lvl, nu, M, p, lvl > 1, rank, world) for lvl, (nu, M) in enumerate(levels, start=1)]
    torch.cuda.synchronize(dev)
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    def step():
        out = runner.run_levels(inputs)
        if world > 1:
            for s in out:
                dist.all_reduce(s)
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    launches0 = _lib.kernel_launches()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush_l2(l2)
            barrier()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            torch.cuda.synchronize(dev)
            barrier()
            times.append(e0.elapsed_time(e1))
    launches = _lib.kernel_launches() - launches0
    # analysis pass (not part of the headline): levels one after another on the main stream, per-level
    # time and per-tier events for the roofline
    runner.records.clear()
    runner.record = True
    level_ms = np.zeros(len(levels))
    apasses = 2
    for ap in range(apasses + 1):  # the first pass warms the main context's buffers
        if ap == 1:
            runner.records.clear()
            level_ms[:] = 0.0
        for li, inp in enumerate(inputs):
            flush_l2(l2)
            torch.cuda.synchronize(dev)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            runner.run_level(inp)
            b.record()
            torch.cuda.synchronize(dev)
            level_ms[li] += a.elapsed_time(b) / apasses
    runner.record = False
    total_ms = float(sum(times))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    total_samples = world * sum(M for _, M in levels)  # weak scaling: every rank runs a full level set
    value = total_samples / (ms_per_step * 1e-3)

    # per-tier accounting for the roofline (algorithmic 16/3 d^3 per (sample, k) matrix)
    tiers = {}
    for rec in runner.records:
        ms = rec["events"][0].elapsed_time(rec["events"][1])
        d = kept_dims(rec["cell"], rec["uniq"])
        flops = float(np.sum(16.0 / 3.0 * d.astype(np.float64) ** 3)) * rec["nk"]
        t = tiers.setdefault(rec["N"], {"N": rec["N"], "ms": 0.0, "flops": 0.0, "matrices": 0, "launches": 0})
        t["ms"] += ms
        t["flops"] += flops
        t["matrices"] += rec["unique"] * rec["nk"]
        t["launches"] += 1
    dom = max(tiers.values(), key=lambda t: t["ms"])
    peak = fp64_peak_live(dev)
    achieved = dom["flops"] / (dom["ms"] * 1e-3) / 1e12
    level_info = []
    for (nu, M), ms in zip(levels, level_ms):
        level_info.append({"nu": nu, "q": nq // nu, "M": M, "ms": round(float(ms), 3),
                           "samples_per_s": round(M / (ms * 1e-3), 2) if ms > 0 else None})

    # e2e through the public Engine API (host buffers, copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(hx, model, levels, nq, p, erange, lo, hi, args, rank, world, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(kind, levels, nq, p, erange)

    if rank == 0:
        line = {
            "metric": "IDOS samples/sec per MLMC level (graphene MLMC, BASELINE config 2)" if args.config == "c2"
            else f"IDOS samples/sec ({desc})",
            "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded reference sampler, bit-exact masks)",
            "config": {"workload": desc, "bz_mode": "reduced (== full to <1e-10, SURVEY finding 3)",
                       "energy_points": NPTS, "delta": DELTA, "master_seed": SEED, "levels": level_info,
                       "l2": "flushed between timed steps (256 MB write)", "parallelism": f"replicas x{world} (rank r draws replicates [r*M, (r+1)*M) of each level stream; one all-reduce of level sums)",
                       "schedule": "all levels and both tiers of each level (parent nu, quarters nu/2) in flight at once on independent streams + contexts; largest tier on a high-priority stream",
                       "levels_note": "per-level ms from a separate sequential analysis pass (the timed step runs them concurrently)"},
            "roofline": {"bound": "fp64", "kernel": f"batched eigensolve N={dom['N']}", "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                         "peak_source": "live cuBLAS ZGEMM 4096^3 complex128 on this GPU (best of 5)",
                         "flops_per_launch": dom["flops"] / max(1, dom["launches"]),
                         "tiers": sorted(tiers.values(), key=lambda t: -t["ms"])},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(hx, model, levels, nq, p, erange, lo, hi, args, rank, world, dev):
    import torch
    import torch.distributed as dist

    plan_levels = levels

    def one(count_bytes):
        eng = hx.Engine(model, nq=nq, delta=DELTA, master_seed=SEED, bz_mode="reduced", energy_points=NPTS,
                        energy_range=(lo + 2 * DELTA, hi - 2 * DELTA), device=dev.index, shard=(rank, world))
        t0 = time.perf_counter()
        for lvl, (nu, M) in enumerate(plan_levels, start=1):
            eng.sample_level(lvl, nu, M, p, with_cv=lvl > 1)
        torch.cuda.synchronize(dev)
        dt = time.perf_counter() - t0
        return dt, eng.io_bytes

    for _ in range(1):
        one(False)
    dts, io = [], None
    for _ in range(max(1, min(args.steps, 3))):
        if world > 1:
            dist.barrier()
        dt, io = one(True)
        dts.append(dt)
    dt = statistics.median(dts)
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    total = world * sum(M for _, M in levels)
    return {"value": total / dt, "unit": "samples/s", "h2d_bytes_per_step": int(io[0]), "d2h_bytes_per_step": int(io[1]),
            "api": "paper_1611_09784_b200.Engine.sample_level per level (host RNG + dedup, hx_eval_idos_batch)"}


def cpu_baseline(kind, levels, nq, p, erange):
    cores = len(os.sched_getaffinity(0))
    frac = 1.0 / 8.0
    try:
        reference_engine_run(kind, levels[:1], nq, p, erange, 16 / levels[0][1], cores)  # warm-up
        per = reference_engine_run(kind, levels, nq, p, erange, frac, cores)
        kindname = "reference"
    except Exception:  # noqa: BLE001 - reference not installed: time the oracle port instead
        return None
    tot_s = sum(x["seconds"] for x in per)
    tot_m = sum(x["M"] for x in per)
    return {"value": tot_m / tot_s, "unit": "samples/s", "cores": cores, "kind": kindname,
            "sample": f"every level with M_l/8 samples through the reference Engine (workers={cores}, reduced BZ)",
            "levels": per}


if __name__ == "__main__":
    sys.exit(main())
