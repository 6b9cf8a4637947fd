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
    # BASELINE config 4: 64 samples sharded over 8 GPUs -> 8 per GPU (weak: each rank its own replicates)
    "c4": ("graphene", [(64, 8)], 128, 0.02, None, "graphene MC nu=64 (N=8192) Gamma+2x2 grid (4 reduced k) p=0.02 M=8/GPU"),
    # BASELINE config 5: batched eigensolve + IDOS sweep, one matrix per (mask, k) (run_c5)
    # (nu1, nu2) supercells: n = 2 nu1 nu2 = 32 ... 2048; the rectangular ones (n = 64, 256, 1024) are this
    # package's n x n2 extension of the reference's square supercells (geometry.build_supercell(n, n2))
    "c5": ("graphene", [(4, 4), (4, 8), (8, 8), (8, 16), (16, 16), (16, 32), (32, 32)], 0, 0.05, None,
           "batched eigensolve+IDOS sweep n=32/64/128/256/512/1024/2048 (graphene-vacancy Bloch matrices, ~50% HBM batches)"),
}
FRAC_NOTE = ("frac = EXECUTED FP64 flops / device time / FP64 peak.  Executed flops are ncu instruction counts of the "
             "same workload and build (DFMA x2 + DMUL + DADD per thread instruction, DMMA m8n8k4 x512 per warp "
             "instruction; tools/ncu_flops.py over a serialised pass, committed under profiles/) - the bipartite SVD, real "
             "arithmetic at time-reversal-invariant k and k/-k pairing mean far fewer flops are executed than the "
             "SURVEY 8(d) count 16/3 d^3 per (sample, k) matrix, which is reported separately as `algorithmic` "
             "(a rate of the dense complex-Hermitian method, not a hardware fraction).")
# executed-FP64 profiles (tools/profile_run.py under ncu + tools/ncu_flops.py --json): config -> path
EXECUTED = {"c2": "profiles/r02_fp64_executed_c2.json", "c3": "profiles/r02_fp64_executed_c3.json",
            "c4": "profiles/r02_fp64_executed_c4.json", "c1": "profiles/r02_fp64_executed_c1.json",
            "c5": "profiles/r02_fp64_executed_c5.json"}
# the dominant tier alone (--levels L --parent-only): (config, N) -> path
EXECUTED_TIER = {("c2", 2048): "profiles/r02_fp64_executed_c2_L4_parent.json",
                 ("c4", 8192): "profiles/r02_fp64_executed_c4.json", ("c1", 32): "profiles/r02_fp64_executed_c1.json"}


def executed_gflop(path):
    """Executed FP64 GFLOP per pass from a committed ncu summary (None when absent)."""
    if path is None or not (ROOT / path).exists():
        return None
    return json.loads((ROOT / path).read_text())["executed_gflop_per_pass"]


# c5 batches: floor(0.5 * 180 GB / (16 n^2)) matrices, one (mask, k) matrix each
C5_BATCH = {32: 5_490_000, 64: 1_370_000, 128: 343_000, 256: 85_800, 512: 21_500, 1024: 5_360, 2048: 1_341}
SEED = 2026
DELTA = 0.01
NPTS = 201


# ncu DRAM bytes (read + write) of one hx_eval_idos_batch_device call of the dominant tier, the same masks
# as the bench's tier (seeded), from a committed capture: (config, N) -> (profile, line prefix)
TRAFFIC = {("c2", 2048): ("profiles/r02_traffic_L4_parent.txt", "total (hx kernels)")}


def traffic_of(config, N):
    """Bytes per launch from the committed ncu summary (None when there is no capture for this tier)."""
    import re

    path, prefix = TRAFFIC.get((config, N), (None, None))
    if path is None or not (ROOT / path).exists():
        return None
    for line in (ROOT / path).read_text().splitlines():
        if line.startswith(prefix):
            m = re.search(r"= ([0-9.]+) GB", line)
            return float(m.group(1)) * 1e9 if m else None
    return None


def env_rank():
    """(rank, world, local device).  HX_BENCH_ONE_DEVICE=1 puts every rank on device 0 - only for the functional
    test of the multi-rank path on a one-GPU box (with HX_DIST_BACKEND=gloo: host-side collectives, the ranks'
    kernels never wait on each other); never for a measurement."""
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if os.environ.get("HX_BENCH_ONE_DEVICE") == "1" else int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


from paper_1611_09784_b200 import _dist  # noqa: E402


def init_dist(local):
    import torch
    import torch.distributed as dist

    backend = os.environ.get("HX_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)


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


REF_MAX_STEPS = 8


def ref_fraction(levels, cores, floor):
    """Sample fraction of the reference legs: the smallest level gets at least `cores` samples (every worker
    busy on every level; c2 on 16 cores: 1/4 -> M = 1024/256/64/16), and at least `floor`."""
    m_min = min(M for _, M in levels)
    return min(1.0, max(floor, cores / m_min))


def host_cpu():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return f"{line.split(':', 1)[1].strip()} x {len(os.sched_getaffinity(0))} threads"
    except OSError:
        pass
    return None


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


LARGE_NU = 64  # levels at or above this size are timed by one reference eigensolve, extrapolated


def reference_single_solve(kind, nu, q, p, cores):
    """Bounded reference sample for the large-N configs (c4: one N = 8192 sample is ~4 x 50 s of LAPACK on
    16 cores): ONE k-point (Gamma) of one seeded sample through the reference's solve_bands + idos
    (spectrum.py:120-134, qoi.py:96-102) with every host core as BLAS threads; per-sample time =
    q^2 x that (the k-points of a sample cost the same).  Returns (seconds per sample, solve seconds)."""
    ref = ROOT / "baseline" / "_ref"
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_hexmc")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import hexmc
    from hexmc.disorder import SeedSpec, sample_defects
    from hexmc.lattice import build_supercell
    from hexmc.qoi import EnergyGrid, SmoothingSpec, idos
    from hexmc.spectrum import make_bz_grid, solve_bands
    from threadpoolctl import threadpool_limits

    model = hexmc.GrapheneNNModel() if kind == "graphene" else hexmc.load_coupling_table(TABLE)
    sc = build_supercell(model.lattice_spec(), nu)
    cfg = sample_defects(sc, p, SeedSpec(SEED, 1, 0))
    grid1 = make_bz_grid(model.lattice_spec(), nu, 1, "reduced")  # Gamma only
    with threadpool_limits(limits=cores):
        sc2 = build_supercell(model.lattice_spec(), 2)  # warm-up (numba kernels, LAPACK threads)
        idos(solve_bands(model, sc2, None, make_bz_grid(model.lattice_spec(), 2, 1, "reduced")),
             EnergyGrid(LO_G, HI_G, NPTS), SmoothingSpec(DELTA), sc2.area)
        t0 = time.perf_counter()
        bands = solve_bands(model, sc, cfg, grid1)
        idos(bands, EnergyGrid(LO_G, HI_G, NPTS), SmoothingSpec(DELTA), sc.area)
        dt = time.perf_counter() - t0
    return dt * q * q, dt


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    kind, levels, nq, p, erange, desc = CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    frac = ref_fraction(levels, cores, args.ref_fraction)
    if max(nu for nu, _ in levels) >= LARGE_NU:
        nu = levels[-1][0]
        try:
            vals = [1.0 / reference_single_solve(kind, nu, nq // nu, p, cores)[0] for _ in range(max(1, args.steps))]
        except Exception as exc:  # noqa: BLE001
            print(json.dumps({"impl": "reference", "unavailable": f"reference import/run failed: {exc!r}"[:300]}))
            return 0
        value = statistics.median(vals)
        sample = (f"one nu={nu} Gamma-point solve_bands+idos per step ({cores} BLAS threads), x{(nq // nu) ** 2} "
                  "k-points per sample (extrapolated)")
        print(json.dumps({"impl": "reference", "metric": f"IDOS samples/sec ({desc})", "value": value,
                          "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": 0,
                          "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded reference sampler)",
                          "config": {"workload": desc}, "cpu_baseline": {"value": value, "unit": "samples/s",
                                                                          "cores": cores, "kind": "reference",
                                                                          "sample": sample},
                          "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return 0
    try:
        # warm-up: one small level (loky spawn + numba load), then timed steps
        for _ in range(max(1, args.warmup)):
            reference_engine_run(kind, levels[:1], nq, p, erange, min(frac, 16 / levels[0][1]), cores)
        step_vals, step_ms, last = [], [], None
        for _ in range(min(args.steps, REF_MAX_STEPS)):
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
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": len(step_vals), "steps_requested": args.steps,
        "warmup": args.warmup,
        "ms_per_step": statistics.median(step_ms), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded reference sampler)", "impl": "reference",
        "config": {"workload": desc, "bz_mode": "reduced", "levels": last, "sample_fraction": frac,
                   "host_cpu": host_cpu(), "same_config": frac == 1.0,
                   "note": f"each step = every level at M_l x {frac:g} (every level >= {cores} samples, so no worker "
                           f"idles); at most {REF_MAX_STEPS} steps so the run stays within a few minutes"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "reference",
                         "sample": f"each step = every level with M_l x {frac} samples, reference Engine "
                                   f"workers={cores} (1 BLAS thread each)"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------------------------------
def c5_reference_sample(kind, nu, words, kp, lo, hi, budget_s=2.0):
    """The reference's own per-matrix path (spectrum.solve_bands + qoi.idos) on host cores, bounded."""
    ref = ROOT / "baseline" / "_ref"
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import hexmc
    from hexmc.disorder import DefectConfiguration
    from hexmc.lattice import build_supercell
    from hexmc.qoi import EnergyGrid, SmoothingSpec, idos
    from hexmc.spectrum import BzGrid, solve_bands

    model = hexmc.GrapheneNNModel()
    sc = build_supercell(model.lattice_spec(), nu)
    grid = BzGrid(n=nu, q=1, mode="reduced", kpoints=np.asarray(kp, dtype=float), weights=np.ones(len(kp)) / len(kp))
    eg = EnergyGrid(lo, hi, NPTS)
    sm = SmoothingSpec(DELTA)
    def solve(row):
        key = int.from_bytes(np.ascontiguousarray(row).tobytes(), "little")
        return idos(solve_bands(model, sc, DefectConfiguration.from_key(sc, key), grid), eg, sm, sc.area)

    solve(words[0])  # warm-up (imports, numba)
    n, t0 = 0, time.perf_counter()
    for row in words:
        solve(row)
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return {"nu": nu, "matrices": n * len(kp), "seconds": time.perf_counter() - t0}


def run_c5(args):
    """Batched eigensolve + IDOS throughput per matrix size (BASELINE config 5): for each n, C5_BATCH[nu]
    seeded graphene-vacancy masks (p = 0.05) at one generic k-point, one hx_eval_idos_batch_device call
    (compaction -> assembly -> eigenvalues -> per-matrix IDOS on the 201-point grid)."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    if world > 1:
        init_dist(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_1611_09784_b200 as hx
    from paper_1611_09784_b200 import _lib
    from paper_1611_09784_b200.device_runner import kept_dims

    kind, levels, _, p, erange, desc = CONFIGS["c5"]
    lo, hi = grid_range(kind, erange)
    model = make_model(kind)
    lib = _lib.load()
    ctx = _lib.Device.ctx(local)
    st = torch.cuda.current_stream(dev)
    g = _lib.EGrid()
    g.e0, g.step, g.npts, g.delta = lo, (hi - lo) / (NPTS - 1), NPTS, DELTA
    peak = fp64_peak_live(dev)
    # executed FP64 per matrix of each size (ncu counts of tools/c5_sample.py batches, profiles/)
    c5_path = ROOT / EXECUTED["c5"]
    c5_exec = json.loads(c5_path.read_text())["per_matrix_gflop"] if c5_path.exists() else {}
    sweep, tot_mats, tot_ms, launches0 = [], 0, 0.0, _lib.kernel_launches()
    e2e_tot = [0, 0.0, 0, 0]  # matrices, seconds, h2d bytes, d2h bytes
    cpu_rows = []
    with ClockSampler(local) as clk:
        for nu, nu2 in levels:
            sc = hx.build_supercell(model.lattice_spec(), nu, nu2)
            cell = hx.compile_cell(model, sc, local)
            nunits = cell.supercell.nunits
            w = max(1, (nunits + 63) // 64)
            B = C5_BATCH[cell.dim]
            masks = torch.zeros((B, w), dtype=torch.int64, device=dev)
            _lib.check(lib.hx_sample_masks_device(SEED, 5, rank * B, B, p, nunits, masks.data_ptr(), st.cuda_stream),
                       "hx_sample_masks_device")
            # one generic k: reduced point (1/3, 1/3) of the supercell zone (the q = 3 grid's point 4 when square)
            b1, b2 = model.lattice_spec().reciprocal_vectors()
            kp = np.ascontiguousarray((b1 / (3 * nu) + b2 / (3 * nu2)).reshape(1, 2))
            curves = torch.empty((B, NPTS), dtype=torch.float64, device=dev)
            status = torch.empty((B, 1), dtype=torch.int32, device=dev)

            def call():
                _lib.check(lib.hx_eval_idos_batch_device(ctx, cell.handle, _lib.ptr(kp), 1, masks.data_ptr(), B,
                                                          C.byref(g), curves.data_ptr(), 0, status.data_ptr(),
                                                          st.cuda_stream), "hx_eval_idos_batch_device")

            for _ in range(args.warmup):
                call()
            torch.cuda.synchronize(dev)
            times = []
            for _ in range(args.steps):
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize(dev)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                call()
                e1.record()
                torch.cuda.synchronize(dev)
                times.append(e0.elapsed_time(e1))
            ms = statistics.median(times)
            if world > 1:
                t = torch.tensor([ms], dtype=torch.float64, device=dev)
                _dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            d = kept_dims(cell, masks)
            flops = float(np.sum(16.0 / 3.0 * d.astype(np.float64) ** 3))
            ach = flops / (ms * 1e-3) / 1e12
            per_mat = c5_exec.get(str(cell.dim))
            exe = None if per_mat is None else per_mat * 1e9 * B / (ms * 1e-3) / 1e12
            if not bool(((status == 0) | (status == 3)).all().item()):
                raise SystemExit(f"c5 n={cell.dim}: failed solves in the timed batch")
            sweep.append({"n": cell.dim, "nu": nu, "nu2": nu2, "batch": B, "ms": round(ms, 3),
                          "matrices_per_s": world * B / (ms * 1e-3), "algorithmic_tflops": round(ach, 3),
                          "executed_tflops": None if exe is None else round(exe, 3),
                          "roofline_frac": None if exe is None else round(exe / peak, 4),
                          "status_ok": True})
            tot_mats += world * B
            tot_ms += ms
            # e2e: the host-buffer API (masks H2D and curves D2H inside the timed region)
            if not args.no_e2e:
                from paper_1611_09784_b200.solver import eval_batch

                hmask = masks.cpu().numpy().view(np.uint64)
                eval_batch(cell, kp, hmask[: min(B, 1024)], lo, g.step, NPTS, DELTA)  # warm
                t0 = time.perf_counter()
                cv, _, _ = eval_batch(cell, kp, hmask, lo, g.step, NPTS, DELTA)
                e2e_s = time.perf_counter() - t0
                sweep[-1]["e2e_matrices_per_s"] = B / e2e_s
                e2e_tot[0] += B
                e2e_tot[1] += e2e_s
                e2e_tot[2] += hmask.nbytes + kp.nbytes
                e2e_tot[3] += cv.nbytes + B * 4
                del hmask, cv
            if rank == 0 and world == 1 and not args.no_cpu_baseline and nu == nu2:  # reference: square cells only
                cpu_rows.append(c5_reference_sample(kind, nu, masks[:64].cpu().numpy().view(np.uint64), kp, lo, hi))
            del masks, curves, status
    launches = _lib.kernel_launches() - launches0
    if rank == 0:
        dom = max(sweep, key=lambda r: r["ms"])
        line = {
            "metric": "batched eigensolve+IDOS matrices/s (BASELINE config 5 sweep)", "value": tot_mats / (tot_ms * 1e-3),
            "unit": "matrices/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded reference sampler, bit-exact masks, p=0.05)",
            "config": {"workload": desc, "sweep": sweep, "k": "one generic reduced-grid k-point per matrix",
                       "energy_points": NPTS, "delta": DELTA},
            "roofline": {"bound": "fp64", "kernel": f"batched eigensolve n={dom['n']} (the sweep's longest batch)",
                         "achieved": dom["executed_tflops"], "peak": peak, "unit": "TFLOP/s",
                         "frac": dom["roofline_frac"], "traffic": None, "executed_source": EXECUTED["c5"],
                         "algorithmic": {"count": "16/3 d^3 per matrix (SURVEY 8d)",
                                         "rate_tflops": dom["algorithmic_tflops"]},
                         "peak_source": "live cuBLAS ZGEMM 4096^3 complex128 on this GPU (best of 5)",
                         "note": FRAC_NOTE},
            "gpu_launches": launches, "clocks": clk.summary(),
            "e2e": None if not e2e_tot[0] else {
                "value": e2e_tot[0] / e2e_tot[1], "unit": "matrices/s", "h2d_bytes_per_step": e2e_tot[2],
                "d2h_bytes_per_step": e2e_tot[3], "api": "solver.eval_batch (hx_eval_idos_batch, host buffers)"},
            "cpu_baseline": None if not cpu_rows else {
                "value": sum(r["matrices"] for r in cpu_rows) / sum(r["seconds"] for r in cpu_rows),
                "unit": "matrices/s", "cores": 1, "kind": "reference",
                "sample": "per n: the reference's solve_bands + idos (zhegv per k, one BLAS thread) on the first "
                          "masks of the same batch, ~2 s each", "per_n": cpu_rows},
        }
        print(json.dumps(line))
    return 0


def spawn_ranks(n):
    """`bench.py --gpus N` run without torchrun: re-launch this command under torch.distributed.run with N
    ranks (one process per GPU, NCCL); rank 0 prints the JSON line."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py")] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)  # ~1.3 s timed region on c2: several clock samples
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hx", choices=["hx", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--ref-fraction", type=float, default=1.0 / 16.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank a full level set of its own replicates (default); strong: one level set, "
                         "its unique masks split over the ranks by sum d^3, curves all-gathered")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.config == "c5":
        return run_c5(args)

    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    if world > 1:
        init_dist(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_1611_09784_b200 as hx
    from paper_1611_09784_b200 import _lib
    from paper_1611_09784_b200.device_runner import DeviceMlmc, kept_dims

    kind, levels, nq, p, erange, desc = CONFIGS[args.config]
    lo, hi = grid_range(kind, erange)
    model = make_model(kind)
    mode = "replicas" if args.scaling == "weak" else "split"
    runner = DeviceMlmc(model, nq, DELTA, SEED, lo, hi, NPTS, device=local,
                        group=dist.group.WORLD if world > 1 else None, mode=mode)

    def barrier():
        if world > 1:
            dist.barrier()

    inputs = [runner.prepare(lvl, nu, M, p, lvl > 1, rank, world) for lvl, (nu, M) in enumerate(levels, start=1)]
    torch.cuda.synchronize(dev)
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    def step():
        return runner.run_levels(inputs)

    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize(dev)
    runner.check_status()  # every (mask, k) solve of the timed workload succeeded
    value_means = [m.cpu().numpy() for m, _ in out]
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
        _dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    # weak: every rank runs a full level set of its own replicates; strong: one level set split over the ranks
    total_samples = (world if mode == "replicas" else 1) * sum(M for _, M in levels)
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
    level_info = []
    for (nu, M), ms in zip(levels, level_ms):
        level_info.append({"nu": nu, "q": nq // nu, "M": M, "ms": round(float(ms), 3),
                           "samples_per_s": round(M / (ms * 1e-3), 2) if ms > 0 else None})

    # e2e through the public Engine API (host buffers, copies inside the timed region)
    e2e, self_check = None, None
    if not args.no_e2e:
        e2e, e2e_means = run_e2e(hx, model, levels, nq, p, erange, lo, hi, args, rank, world, dev)
        # the timed device pipeline and the public Engine API must give the same level means (same masks,
        # same curves, exact moments): bitwise, for any number of ranks
        diffs = [float(np.max(np.abs(a - b))) for a, b in zip(value_means, e2e_means)]
        self_check = {"level_means_max_abs_diff_vs_engine": max(diffs),
                      "bitwise_equal": all(np.array_equal(a, b) for a, b in zip(value_means, e2e_means))}
        if max(diffs) > 1e-9:
            raise SystemExit(f"self-check failed: device pipeline vs Engine level means differ by {max(diffs)}")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(kind, levels, nq, p, erange)

    if rank == 0:
        line = {
            "metric": "IDOS samples/sec per MLMC level (graphene MLMC, BASELINE config 2)" if args.config == "c2"
            else f"IDOS samples/sec ({desc})",
            "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded reference sampler, bit-exact masks)",
            "config": {"workload": desc, "bz_mode": "reduced (== full to <1e-10, SURVEY finding 3)",
                       "energy_points": NPTS, "delta": DELTA, "master_seed": SEED, "levels": level_info,
                       "l2": "flushed between timed steps (256 MB write)", "parallelism": (f"replicas x{world} (rank r draws replicates [r*M, (r+1)*M) of each level stream; exact fixed-point level sums, int64 all-reduce)" if mode == "replicas" else f"split x{world} (one level set; unique masks of each tier split over the ranks by sum d^3, curves all-gathered)"),
                       "schedule": "all levels and both tiers of each level (parent nu, quarters nu/2) in flight at once on independent streams + contexts; largest tier on a high-priority stream; unique masks per tier (torch.unique on the device), tiers of the same one-word cell deduplicated together (the reference run cache's cross-level hits, runner.py:213-233)",
                       "levels_note": "per-level ms from a separate sequential analysis pass (the timed step runs them concurrently)"},
            "roofline": roofline_block(args.config, world, mode, ms_per_step, peak, dom, tiers, apasses),
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "e2e": e2e,
            "self_check": self_check,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def roofline_block(config, world, mode, ms_per_step, peak, dom, tiers, apasses):
    """FP64 roofline of the timed step: executed flops (ncu counts of the same pass) / device time / peak; the
    dominant tier (largest event time in the sequential analysis pass) likewise; the SURVEY 8(d) algorithmic
    count reported beside it as a rate, not a fraction."""
    per_rank_sets = 1 if mode == "replicas" else 1.0 / world  # level sets a rank runs per step
    exe = executed_gflop(EXECUTED.get(config))
    achieved = None if exe is None else exe * 1e9 * per_rank_sets / (ms_per_step * 1e-3) / 1e12
    block = {"bound": "fp64", "kernel": f"batched eigensolve, every hx kernel of one {config} step (all tiers)",
             "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
             "frac": None if achieved is None else achieved / peak,
             "executed_gflop_per_step": None if exe is None else exe * per_rank_sets,
             "executed_source": EXECUTED.get(config),
             "peak_source": "live cuBLAS ZGEMM 4096^3 complex128 on this GPU (best of 5)", "note": FRAC_NOTE}
    tier_exe = executed_gflop(EXECUTED_TIER.get((config, dom["N"])))
    dom_ms = dom["ms"] / max(1, dom["launches"])
    block["dominant_tier"] = {
        "N": dom["N"], "ms_per_launch": dom_ms, "matrices_per_launch": dom["matrices"] / max(1, dom["launches"]),
        "executed_gflop_per_launch": tier_exe, "executed_source": EXECUTED_TIER.get((config, dom["N"])),
        "achieved_tflops": None if tier_exe is None else tier_exe / dom_ms,
        "frac": None if tier_exe is None else tier_exe / dom_ms / peak,
        "traffic": traffic_of(config, dom["N"]), "traffic_source": TRAFFIC.get((config, dom["N"]), (None, None))[0]}
    block["traffic"] = block["dominant_tier"]["traffic"]
    alg = sum(t["flops"] for t in tiers.values()) / apasses
    block["algorithmic"] = {"count": "16/3 d^3 per (sample, k) matrix solved (SURVEY 8d)", "flops_per_step": alg,
                            "rate_tflops": alg * per_rank_sets / (ms_per_step * 1e-3) / 1e12,
                            "note": "matrices of the sequential analysis pass (every tier deduplicated on its own); the "
                                    "timed step deduplicates same-cell one-word tiers together (the reference run "
                                    "cache's cross-level hits) and solves ~20 % fewer nu = 4 matrices: ~0.1 % of "
                                    "these flops on c2"}
    block["tiers"] = sorted(tiers.values(), key=lambda t: -t["ms"])
    return block


def run_e2e(hx, model, levels, nq, p, erange, lo, hi, args, rank, world, dev):
    """Engine.run_mlmc (the public API) with host buffers; returns (e2e dict, level means of the last run)."""
    import torch
    import torch.distributed as dist

    plan_levels = levels
    shard_mode = "replicas" if args.scaling == "weak" else "split"

    def one(count_bytes):
        eng = hx.Engine(model, nq=nq, delta=DELTA, master_seed=SEED, bz_mode="reduced", energy_points=NPTS,
                        energy_range=(lo + 2 * DELTA, hi - 2 * DELTA), device=dev.index, shard=(rank, world),
                        shard_mode=shard_mode)
        plan = hx.LevelPlan(ns=tuple(nu for nu, _ in plan_levels), samples=tuple(M for _, M in plan_levels), nq=nq,
                            p_vac=p, delta=DELTA)
        t0 = time.perf_counter()
        _, sets = eng.run_mlmc(plan)
        torch.cuda.synchronize(dev)
        dt = time.perf_counter() - t0
        return dt, eng.io_bytes, [s.stats.mean for s in sets]

    for _ in range(1):
        one(False)
    dts, io = [], None
    for _ in range(max(1, min(args.steps, 3))):
        if world > 1:
            dist.barrier()
        dt, io, means = one(True)
        dts.append(dt)
    dt = statistics.median(dts)
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        _dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    total = (world if shard_mode == "replicas" else 1) * sum(M for _, M in levels)
    return {"value": total / dt, "unit": "samples/s", "h2d_bytes_per_step": int(io[0]), "d2h_bytes_per_step": int(io[1]),
            "api": f"paper_1611_09784_b200.Engine.run_mlmc (shard_mode={shard_mode}; masks drawn on the GPU and read back (rng='device', bit-identical to the host sampler), host dedup / cache / placement per level, every (n, q) tier of every level through hx_eval_idos_batch with host buffers, concurrently)"}, means


def cpu_baseline(kind, levels, nq, p, erange):
    cores = len(os.sched_getaffinity(0))
    frac = ref_fraction(levels, cores, 1.0 / 16.0)
    if max(nu for nu, _ in levels) >= LARGE_NU:
        nu = levels[-1][0]
        try:
            per_sample, solve_s = reference_single_solve(kind, nu, nq // nu, p, cores)
        except Exception:  # noqa: BLE001 - reference not installed
            return None
        return {"value": 1.0 / per_sample, "unit": "samples/s", "cores": cores, "kind": "reference",
                "sample": f"one nu={nu} Gamma-point solve_bands+idos of a seeded sample ({solve_s:.1f} s, {cores} BLAS "
                          f"threads), x{(nq // nu) ** 2} k-points per sample (extrapolated)"}
    try:
        reference_engine_run(kind, levels[:1], nq, p, erange, 16 / levels[0][1], cores)  # warm-up
        per = reference_engine_run(kind, levels, nq, p, erange, frac, cores)
        kindname = "reference"
    except Exception:  # noqa: BLE001 - reference not installed: time the oracle port instead
        return None
    tot_s = sum(x["seconds"] for x in per)
    tot_m = sum(x["M"] for x in per)
    return {"value": tot_m / tot_s, "unit": "samples/s", "cores": cores, "kind": kindname,
            "sample": f"every level with M_l x {frac:g} samples through the reference Engine (workers={cores}, reduced "
                      f"BZ; every level >= {cores} samples)", "host_cpu": host_cpu(), "levels": per}


if __name__ == "__main__":
    sys.exit(main())
