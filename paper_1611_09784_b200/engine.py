"""Run orchestration on the GPU backend: the drop-in for the reference Engine (runner.py:148-439).

The reference's batch seam `evaluate_masks -> parallel_map(_eval_job, jobs)` (runner.py:206-244) is
kept with identical dedup/placement semantics (key (n, q, mask), run-wide cache shared across levels
and CV quarters, in-batch owners), but the new jobs of each (n, q) group go to ONE libhx batch call
(hx_eval_idos_batch) instead of a process pool.  Sampling (bit-exact with numpy), quarter restriction
and level moments run in libhx as well.  Results do not depend on batch composition (fixed-point
IDOS accumulation), so curves are identical for any grouping of requests.

BZ mode "full" is evaluated on its q^2 base points with weights 1/q^2: the two rotated rhombi are
periodic images of the base grid point for point (spectrum.py:8-14), so the quadrature is the same and
curves agree with the reference's full mode to rounding (SURVEY finding 3; pinned by
tests/test_fx_gpu.py against the reference's full-mode fixtures).

Several GPUs, results bitwise identical to one GPU (the reference's "identical for any worker
count", /root/reference/pkg/tests/test_runner.py:39-43):
  Engine(devices=G)          one process, the new unique masks of every (n, q) group split over G devices in
                             contiguous slices balanced by sum d^3 (d = kept dimension); cache semantics and
                             cache_hits are the single-device ones (the dedup is unchanged).
  Engine(shard=(rank, world)) one process per GPU under torch.distributed: rank r draws the replicates
                             [r*M, (r+1)*M) of each level stream and the level moments are combined exactly
                             (fixed-point limbs, int64 all-reduce): the mean / variance bits of one process
                             drawing world*M replicates.  cache_hits are per rank.
  Engine(shard=(rank, world), shard_mode="split")  one process per GPU, strong scaling: every rank draws the
                             whole level, dedups it identically and solves its d^3-balanced slice of each
                             group's new masks; the slices' curves are all-gathered, so every rank holds the
                             single-process results (curves, moments and cache_hits bit for bit).
"""

from __future__ import annotations

import functools
import math
import os
import threading
import time
from concurrent.futures import FIRST_COMPLETED, ThreadPoolExecutor, wait
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .estimators import (LevelPlan, LevelStats, RateEstimates, combine_levels, exact_level_moments,
                         fit_rates, level_moments, mean_and_variance, window_mask)
from .geometry import build_supercell, partition_quarters
from .idos import EnergyGrid
from .models import compile_cell
from .sampling import (DefectConfiguration, enumerate_configs, keys_from_words, restrict_words, sample_masks,
                       words_from_keys)
from .solver import (eval_batch, make_bz_grid, raise_status, solve_bands, time_reversal_reduce,
                     use_time_reversal)

__all__ = ["Engine", "TaskError", "LevelSampleSet", "ExhaustiveResult", "RatesResult", "SLMC_STREAM_OFFSET"]

SLMC_STREAM_OFFSET = 10_000

# Compiled cells (device-resident instance tables) shared by every Engine of the process, keyed on the
# (hashable, frozen) model, the supercell size and the device: the reference keeps the same per-process
# cache in each worker (runner.py:98-111).  Rebuilding them per Engine costs a few ms of uploads, and
# releasing them (cudaFree) synchronises the device.
_CELL_CACHE: dict = {}
# k-point sets (and their time-reversal reduction) per (lattice, n, q): process-wide like the cells
_KGRID_CACHE: dict = {}
# Concurrent tier schedule of the seam: the largest tier is planned and submitted first (it is the critical
# path), then the others smallest first; the small tiers (dim <= 128) run on the greatest stream priority so
# that their levels finish early and the host work of placing them overlaps the device work still running,
# the largest tier next, the rest at the default priority (e2e run_mlmc on c2: 87 -> 71 ms with pinned
# staging).  Experiments: HX_E2E_PRIO=big|big+small, HX_E2E_ORDER=big-first.
_E2E_PRIO = os.environ.get("HX_E2E_PRIO", "tiered")
_E2E_ORDER = os.environ.get("HX_E2E_ORDER", "big-then-small")
_E2E_WORKERS = int(os.environ.get("HX_E2E_WORKERS", "4"))  # concurrent (tier, level) pieces (0: all at once); c2 e2e 121k (all 7) -> 127k


def unique_rows(words):
    """np.unique(words, axis=0, return_inverse=True) for uint64 mask rows - the same lexicographic order -
    without the structured-array path of axis=0 (10x faster on the seam's 4096-row tiers)."""
    R, w = words.shape
    if w == 1:
        u, inv = np.unique(words[:, 0], return_inverse=True)
        return u.reshape(-1, 1), inv.reshape(-1)
    if R == 0:
        return words[:0], np.zeros(0, dtype=np.int64)
    order = np.lexsort(words.T[::-1])  # column 0 is the primary key
    srt = words[order]
    new = np.empty(R, dtype=bool)
    new[0] = True
    new[1:] = np.any(srt[1:] != srt[:-1], axis=1)
    inv = np.empty(R, dtype=np.int64)
    inv[order] = np.cumsum(new) - 1
    return srt[new], inv


def first_rows(inv):
    """Index of the first occurrence of each value 0..max(inv) in inv (every value occurs)."""
    if len(inv) == 0:
        return np.zeros(0, dtype=np.int64)
    return np.unique(inv, return_index=True)[1]


_RNG_STREAMS: dict = {}
_QMAPS: dict = {}


def _rng_stream(device):
    import torch

    st = _RNG_STREAMS.get(device)
    if st is None:
        st = _RNG_STREAMS[device] = torch.cuda.Stream(device=device, priority=-1)
    return st


def _quarter_maps(part, device):
    """Device copies of a partition's quarter labels and unit map (cached per parent cell)."""
    import torch

    key = (part.parent.spec, part.parent.n, device)
    if key not in _QMAPS:
        dev = torch.device("cuda", device)
        _QMAPS[key] = (torch.from_numpy(part.unit_assignment.astype(np.int32)).to(dev),
                       torch.from_numpy(part.unit_map.astype(np.int32)).to(dev))
    return _QMAPS[key]


class _InlineExecutor:
    """Executor interface that runs the submitted call immediately (single-piece batches)."""

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False

    def submit(self, fn, *args, **kw):
        from concurrent.futures import Future

        f = Future()
        try:
            f.set_result(fn(*args, **kw))
        except BaseException as exc:  # noqa: BLE001 - delivered through the future like a pool would
            f.set_exception(exc)
        return f


class _TierCache:
    """Run cache of one (n, q) tier: the (n, q, mask) keys of the reference's cache (runner.py:206-244) as a
    sorted array of mask rows (void view of the uint64 words) with the row of each key's curve in an append-only
    buffer, so lookups and inserts are vectorised (searchsorted) and an insert copies only the new curves
    (the buffer grows by doubling; only the small key / index arrays are re-sorted)."""

    def __init__(self, npts):
        self.keys = None
        self.rows = np.zeros(0, dtype=np.int64)
        self.buf = np.zeros((0, npts))
        self.pjb = np.zeros(0)
        self.n = 0

    def find(self, kv):
        """Buffer row of each key, -1 if absent."""
        if self.keys is None or not len(self.keys) or not len(kv):
            return np.full(len(kv), -1, dtype=np.int64)
        pos = np.minimum(np.searchsorted(self.keys, kv), len(self.keys) - 1)
        return np.where(self.keys[pos] == kv, self.rows[pos], -1)

    @property
    def curves(self):
        return self.buf

    @property
    def pj(self):
        return self.pjb

    def add(self, kv, curves, pj):
        k = len(kv)
        if self.n + k > len(self.buf):
            cap = max(2 * len(self.buf), self.n + k, 256)
            nb = np.empty((cap, self.buf.shape[1]))
            nb[: self.n] = self.buf[: self.n]
            npj = np.empty(cap)
            npj[: self.n] = self.pjb[: self.n]
            self.buf, self.pjb = nb, npj
        self.buf[self.n: self.n + k] = curves
        self.pjb[self.n: self.n + k] = pj
        rows = np.arange(self.n, self.n + k)
        self.n += k
        keys = kv if self.keys is None else np.concatenate([self.keys, kv])
        allrows = rows if self.keys is None else np.concatenate([self.rows, rows])
        o = np.argsort(keys, kind="stable")
        self.keys, self.rows = keys[o], allrows[o]

    def __len__(self):
        return self.n


class TaskError(RuntimeError):
    """One or more tasks failed; message names the task ids (runner.py:56-72)."""

    def __init__(self, failures):
        self.failures = failures
        names = ", ".join(str(tid) for tid, _ in failures[:4])
        more = "" if len(failures) <= 4 else f" (+{len(failures) - 4} more)"
        super().__init__(f"{len(failures)} task(s) failed: {names}{more}; first error: {failures[0][1]!r}")


@dataclass(frozen=True, eq=False)
class LevelSampleSet:
    stats: LevelStats
    terms: np.ndarray = field(repr=False)
    full: np.ndarray = field(repr=False)
    cv: np.ndarray | None = field(repr=False, default=None)


@dataclass(frozen=True, eq=False)
class RatesResult:
    records: list
    rates: RateEstimates
    bias_proxies: list


@dataclass(frozen=True, eq=False)
class ExhaustiveResult:
    mean: np.ndarray = field(repr=False)
    variance: np.ndarray = field(repr=False)
    weight_sum: float = 1.0
    nconfigs: int = 0
    evaluations: int = 0
    cache_hits: int = 0
    wall_seconds: float = 0.0
    n: int = 1
    q: int = 1


class Engine:
    """Shared context of one run: model, grids, dedup cache, device (runner.py:148-175)."""

    def __init__(self, model, nq: int, delta: float, master_seed: int, workers: int = 1, bz_mode: str = "full",
                 energy_points: int = 4096, energy_range=None, dedup: bool = True, device: int = 0,
                 shard=(0, 1), devices=1, shard_mode: str = "replicas", rng: str = "device"):
        self.model = model
        self.nq = nq
        self.delta = delta
        self.master_seed = master_seed
        self.workers = workers  # accepted for API parity; the GPU batch replaces the process pool
        self.bz_mode = bz_mode
        self.dedup = dedup
        self.device = device
        self.shard = shard  # (rank, world): rank r draws replicates [r*M, (r+1)*M) (weak-scaling replicas)
        if isinstance(devices, int):
            if devices < 1:
                raise ValueError("devices must be >= 1")
            devices = [device + g for g in range(devices)]
        if shard_mode not in ("replicas", "split"):
            raise ValueError(f"unknown shard mode {shard_mode!r}")
        self.shard_mode = shard_mode
        if rng not in ("device", "host"):
            raise ValueError(f"unknown rng {rng!r}")
        self.rng = rng  # where the level masks are drawn (bit-identical either way)
        self.devices = list(devices)  # GPUs the new masks of a group are split over (int G: device .. device+G-1)
        self.io_bytes = [0, 0]  # host->device, device->host bytes moved by the batch calls
        self._caches: dict = {}  # (n, q) -> _TierCache: the run-wide dedup cache (runner.py:206-244)
        self._coll = threading.Condition()  # split mode: all-gathers in submission order on every rank
        self._coll_turn = 0
        self._coll_tickets = 0
        self._supercells: dict = {}
        self._cells: dict = {}
        if energy_range is None:
            emin, emax = self.detect_energy_range()
        else:
            emin, emax = energy_range
            if not emax > emin:
                raise ValueError("energy range needs max > min")
        self.grid = EnergyGrid(emin - 2.0 * delta, emax + 2.0 * delta, energy_points)

    # -- geometry / caches --
    def supercell(self, n: int):
        if n not in self._supercells:
            key = ("sc", self.model.lattice_spec(), n)
            if key not in _KGRID_CACHE:
                _KGRID_CACHE[key] = build_supercell(self.model.lattice_spec(), n)
            self._supercells[n] = _KGRID_CACHE[key]
        return self._supercells[n]

    def quarters(self, sc):
        """partition_quarters(sc), cached process-wide like the supercells (the nu = 32 partition costs ~1 ms of
        host time, on the critical path of run_mlmc's first submission)."""
        key = ("part", sc.spec, sc.n)
        if key not in _KGRID_CACHE:
            _KGRID_CACHE[key] = partition_quarters(sc)
        return _KGRID_CACHE[key]

    def cell(self, n: int, device: int | None = None):
        device = self.device if device is None else device
        if (n, device) not in self._cells:
            try:
                key = (self.model, n, device)
                hash(key)
            except TypeError:
                key = None
            if key is not None and key in _CELL_CACHE:
                self._cells[(n, device)] = _CELL_CACHE[key]
            else:
                self._cells[(n, device)] = compile_cell(self.model, self.supercell(n), device)
                if key is not None:
                    _CELL_CACHE[key] = self._cells[(n, device)]
        return self._cells[(n, device)]

    def kpoints(self, n: int, q: int) -> np.ndarray:
        """k-points solved for (n, q): the base q x q rhombus (full mode's rotated copies are images)."""
        key = (self.model.lattice_spec(), n, q)
        if key not in _KGRID_CACHE:
            _KGRID_CACHE[key] = make_bz_grid(self.model.lattice_spec(), n, q, "reduced").kpoints
        return _KGRID_CACHE[key]

    def kpoints_tr(self, n: int, q: int):
        """(k-points, multiplicities) of the IDOS batches: time-reversal pairs merged for real-amplitude
        models (solver.time_reversal_reduce), otherwise the full base grid with multiplicity 1."""
        tr = use_time_reversal() and self.cell(n).time_reversal_symmetric
        key = ("tr", self.model.lattice_spec(), n, q, tr)
        if key not in _KGRID_CACHE:
            kp = self.kpoints(n, q)
            _KGRID_CACHE[key] = time_reversal_reduce(self.model.lattice_spec(), n, kp) if tr else (kp, None)
        return _KGRID_CACHE[key]

    def q_of(self, n: int) -> int:
        if self.nq % n:
            raise ValueError(f"n*q constant {self.nq} is not divisible by n = {n}")
        return self.nq // n

    def detect_energy_range(self):
        """Unperturbed nu=1 band range on the shared folded grid (runner.py:189-202)."""
        grid = make_bz_grid(self.model.lattice_spec(), 1, self.nq, self.bz_mode)
        bands = solve_bands(self.model, self.supercell(1), None, grid, cell=self.cell(1))
        return float(bands.energies.min()), float(bands.energies.max())

    def _tier_cache(self, tier, npts):
        c = self._caches.get(tier)
        if c is None:
            c = self._caches[tier] = _TierCache(npts)
        return c

    # -- the batch seam --
    def _solve_split(self, n: int, q: int, words, task_ids, lane: int, high, ticket: int = 0):
        """The new masks of one (n, q) group over self.devices: contiguous slices balanced by sum d^3 (d = kept
        dimension), one thread + context per device; curves in row order (each curve is independent of the
        batch it was solved in, so the split does not change a bit)."""
        rank, world = self.shard
        if world > 1 and self.shard_mode == "split":
            return self._solve_ranks(n, q, words, task_ids, lane, high, ticket)
        G = len(self.devices)
        if G == 1 or len(words) < G:
            ctx = _lib.Device.lane(self.device, lane, high) if lane is not None else None
            return self._solve_group(n, q, words, task_ids, ctx)
        cuts = self._cuts(n, words, G)
        with ThreadPoolExecutor(max_workers=G) as ex:
            # one context per slice (a context serves one host thread at a time; the same GPU may be listed
            # more than once)
            futs = [ex.submit(self._solve_group, n, q, words[a:b], task_ids[a:b],
                              _lib.Device.lane(dev, (lane or 0) * G + g, high), dev)
                    for g, (dev, a, b) in enumerate(zip(self.devices, cuts[:-1], cuts[1:])) if b > a]
            parts = [f.result() for f in futs]
        curves = np.concatenate([cu for cu, _ in parts])
        per_job = sum(pj * len(cu) for cu, pj in parts) / max(1, len(curves))
        return curves, per_job

    def _cuts(self, n, words, parts):
        """Contiguous slices of the rows with equal shares of sum d^3 (the eigensolve cost)."""
        d = self.cell(n).kept_dims(words).astype(np.float64)
        c = np.cumsum(d * d * d)
        cuts = np.concatenate([[0], np.searchsorted(c, c[-1] * np.arange(1, parts) / parts) + 1, [len(words)]])
        return np.maximum.accumulate(np.minimum(cuts, len(words)))

    def _solve_ranks(self, n, q, words, task_ids, lane, high, ticket):
        """shard_mode="split": this rank's d^3-balanced slice of the group's new masks, then an all-gather of
        the slices' curves (NCCL on the device), so every rank returns the whole group in row order."""
        import torch
        import torch.distributed as dist

        rank, world = self.shard
        cuts = self._cuts(n, words, world)
        a, b = int(cuts[rank]), int(cuts[rank + 1])
        ctx = _lib.Device.lane(self.device, lane, high) if lane is not None else None
        npts = self.grid.npoints
        if b > a:
            curves, per_job = self._solve_group(n, q, words[a:b], task_ids[a:b], ctx)
        else:
            curves, per_job = np.zeros((0, npts)), 0.0
        width = int(max(cuts[1:] - cuts[:-1]))
        # the gather runs where the backend lives: device memory for NCCL, host memory for gloo
        dev = torch.device("cuda", self.device) if dist.get_backend() == "nccl" else torch.device("cpu")
        pad = torch.zeros((width, npts + 1), dtype=torch.float64, device=dev)
        pad[: b - a, :npts] = torch.from_numpy(curves).to(dev)
        pad[:, npts] = per_job
        out = torch.empty((world * width, npts + 1), dtype=torch.float64, device=dev)
        with self._coll:  # the collectives of the process group in submission order (the same on every rank)
            self._coll.wait_for(lambda: self._coll_turn == ticket)
            try:
                dist.all_gather_into_tensor(out, pad)
            finally:
                self._coll_turn += 1
                self._coll.notify_all()
        out = out.cpu().numpy()
        rows = np.concatenate([out[r * width: r * width + int(cuts[r + 1] - cuts[r])] for r in range(world)])
        self.io_bytes[0] += (world - 1) * pad.numel() * 8
        return rows[:, :npts].copy(), float(rows[:, npts].mean()) if len(rows) else 0.0

    def _solve_group(self, n: int, q: int, words, task_ids, ctx=None, device=None):
        """One GPU batch for the (n, q) group: words uint64 [R, w] (task_ids: R ids for error reports)."""
        cell = self.cell(n, device)
        kp, kmult = self.kpoints_tr(n, q)
        t0 = time.perf_counter()
        curves, _, status = eval_batch(cell, kp, words, self.grid.lo, self.grid.step, self.grid.npoints,
                                       self.delta, ctx=ctx, kmult=kmult)
        secs = time.perf_counter() - t0
        self.io_bytes[0] += words.nbytes + kp.nbytes
        self.io_bytes[1] += curves.nbytes + status.nbytes
        bad = np.flatnonzero(((status == _lib.HX_ST_NOT_PD) | (status == _lib.HX_ST_NONFINITE)).any(axis=1))
        if len(bad):
            failures = []
            for i in bad:
                try:
                    raise_status(status[i:i + 1], kp)
                except Exception as exc:  # noqa: BLE001 - collected with the task id
                    failures.append((task_ids[i], exc))
            raise TaskError(failures)
        return curves, secs / max(1, len(words))

    def _evaluate_words(self, groups, task_ids):
        """One batch of the seam (see _evaluate_batches)."""
        return self._evaluate_batches([(groups, task_ids)])[0]

    def _evaluate_batches(self, batches, on_batch=None, tiers_of=None):
        """Vectorised batch seam for several consecutive batches.  batches: list of (groups, task_ids),
        groups = [(n, q, words uint64 [R, w]), ...] in request order, task_ids(i_group, new, inv) -> ids of
        the new masks (error reports only).  Every batch is deduplicated on (n, q, mask) against the run
        cache, against itself (np.unique over the rows instead of a per-request dict) and against the new
        masks of the EARLIER batches - the hit accounting of calling the batches one after another
        (runner.py:206-244).  Keys of different (n, q) never meet, so the planning runs one (n, q) tier at
        a time, most expensive tier first, and the new masks each batch contributes to a tier are submitted
        as their own GPU batch (own thread and hx context; the first tier's on the high-priority one) as
        soon as they are planned: the host work of the smaller tiers overlaps the device work of the big
        one, and the pieces of different levels run concurrently.  Returns per batch ([(curves [R, npts],
        per_job [R]) per group], hits, spent).

        A batch may also be given as a zero-argument callable returning (groups, task_ids), with `tiers_of`
        naming the (n, q) of its groups in order: it is then drawn only when the first tier it contributes
        to is planned, so the largest tier's masks are drawn and submitted before the other levels' masks
        exist (the GPU starts while the host is still drawing)."""
        npts = self.grid.npoints
        made: dict = {}

        def get(bi):
            b = batches[bi]
            if callable(b):
                if bi not in made:
                    made[bi] = b()
                return made[bi]
            return b

        if tiers_of is None:
            tiers_of = [[(n, q) for n, q, _w in get(bi)[0]] for bi in range(len(batches))]
        tiers: dict = {}  # (n, q) -> [batch indices contributing] in batch order
        for bi, tl in enumerate(tiers_of):
            for t in tl:
                tiers.setdefault(t, []).append(bi)

        def members(tier):  # [(batch index, group index, words)] of a tier, drawing its batches on demand
            out = []
            for bi in tiers[tier]:
                for gi, (n, q, words) in enumerate(get(bi)[0]):
                    if (n, q) == tier:
                        out.append((bi, gi, np.ascontiguousarray(words, dtype=np.uint64)))
            return out

        for n, q in tiers:
            for dev in self.devices:
                self.cell(n, dev)  # compile cells and k-sets up front (not thread-safe)
            self.kpoints_tr(n, q)
        order = sorted(tiers, key=lambda g: -self.cell(g[0]).dim)
        if _E2E_ORDER == "big-then-small" and len(order) > 2:
            # the largest tier first (critical path), then the rest smallest first
            order = order[:1] + order[1:][::-1]
        elif _E2E_ORDER == "big2-then-small" and len(order) > 3:
            # experiment: the two largest tiers first, then the rest smallest first.  The GPU phase of c2 ends 1.2 ms
            # earlier, but the level-moment kernels of the small levels then queue behind the resident chase CTAs of
            # the large tiers (they hold every register of their SMs for ~4 ms each): level 1's finish waits 24 ms
            # and the host work of the small levels piles up after the GPU is done - e2e 109k vs 138k samples/s
            order = order[:2] + order[2:][::-1]
        hits = [0] * len(batches)
        spent = [0.0] * len(batches)
        plans = {}  # (bi, gi) -> (tier, uniq, inv, keys, src)
        pieces = {}  # tier -> [(first new row, future)] in row order
        lane = 0
        npieces = sum(len(v) for v in tiers.values())
        # one piece (a single-level run): solve it inline, without a thread pool
        nworkers = max(1, min(npieces, _E2E_WORKERS) if _E2E_WORKERS > 0 else npieces)
        with (_InlineExecutor() if npieces == 1 else ThreadPoolExecutor(max_workers=nworkers)) as ex:
            for tier in order:
                cache = self._tier_cache(tier, npts)
                pend = np.zeros(0, dtype=np.int64)  # sorted keys of this call's new masks so far, their rows
                pend_keys = None
                count = 0
                for bi, gi, words in members(tier):
                    R = words.shape[0]
                    start = count
                    if self.dedup and R:
                        uniq, inv = unique_rows(words)
                        kv = uniq.view(f"V{8 * uniq.shape[1]}").ravel()
                        src = np.where(cache.find(kv) >= 0, -1, -2)
                        if pend_keys is not None and len(pend_keys):
                            pos = np.minimum(np.searchsorted(pend_keys, kv), len(pend_keys) - 1)
                            inp = (pend_keys[pos] == kv) & (src == -2)
                            src[inp] = pend[pos[inp]]
                        fresh = np.flatnonzero(src == -2)
                        src[fresh] = count + np.arange(len(fresh))
                        count += len(fresh)
                        if len(fresh):  # fresh rows join the pending set (kept sorted)
                            allk = kv[fresh] if pend_keys is None else np.concatenate([pend_keys, kv[fresh]])
                            allr = src[fresh] if pend_keys is None else np.concatenate([pend, src[fresh]])
                            o = np.argsort(allk, kind="stable")
                            pend_keys, pend = allk[o], allr[o]
                    else:
                        uniq, inv, kv = words, np.arange(R), None
                        src = count + np.arange(R)
                        count += R
                    new = np.flatnonzero(src >= start)
                    hits[bi] += R - len(new)
                    if len(new):
                        ids = get(bi)[1](gi, new, inv)
                        small = self.cell(tier[0]).dim <= 128
                        if _E2E_PRIO == "tiered":
                            # small tiers first (their levels finish early and the host work of placing
                            # them overlaps the device work left), then the largest tier, then the rest
                            high = -100 if small else (-1 if lane == 0 else 0)
                        else:
                            high = lane == 0 or (_E2E_PRIO == "big+small" and small)
                        ln = lane if len(tiers) > 1 or len(tiers[tier]) > 1 else None
                        lane += 1
                        ticket = self._coll_tickets
                        self._coll_tickets += 1
                        pieces.setdefault(tier, []).append(
                            (start, ex.submit(self._solve_split, tier[0], tier[1], uniq[new], ids, ln, high, ticket),
                             bi))
                    plans[(bi, gi)] = (tier, uniq, inv, kv, src, start)
            # group gi of batch bi can be placed once every piece of its tier submitted by batches <= bi is
            # done; groups are placed (curves gathered, run cache filled) as soon as that holds and a batch is
            # finished (on_batch) when its last group is in, so the host work overlaps the device work still
            # running - at the end only the groups of the last tier to finish remain
            needs = {}
            for bi, tl in enumerate(tiers_of):
                for gi, (n, q) in enumerate(tl):
                    needs[(bi, gi)] = [f for (start, f, pbi) in pieces.get((n, q), []) if pbi <= bi]
            out = [None] * len(batches)
            placed = {bi: [None] * len(tl) for bi, tl in enumerate(tiers_of)}
            left = list(needs)
            while left:
                ready = [key for key in left if all(f.done() for f in needs[key])]
                if not ready:
                    wait([f for key in left for f in needs[key] if not f.done()], return_when=FIRST_COMPLETED)
                    continue
                for bi, gi in ready:
                    placed[bi][gi] = self._place_group(bi, gi, plans, pieces, spent, npts)
                    left.remove((bi, gi))
                    if all(r is not None for r in placed[bi]):
                        out[bi] = (placed[bi], hits[bi], spent[bi])
                        if on_batch is not None:
                            on_batch(bi, out[bi])
        return out

    def _place_group(self, bi, gi, plans, pieces, spent, npts):
        """Per-request curves of group gi of batch bi from the run cache and the solved pieces
        (runner.py:234-243).  Every request row is gathered once from its source (a solved piece or the cache) -
        no intermediate array of the unique masks' curves."""
        tier, uniq, inv, kv, src, start = plans[(bi, gi)]
        R = len(inv)
        out = np.empty((R, npts))
        opj = np.empty(R)
        rsrc = src[inv]  # per request row: piece row (>= 0) or cached (< 0)
        pj_u = np.empty(len(uniq))
        got = np.flatnonzero(src >= 0)
        if len(got):
            lst = pieces[tier]
            starts = np.array([st for st, _, _ in lst])
            which_u = np.searchsorted(starts, src[got], side="right") - 1
            which_r = np.searchsorted(starts, rsrc, side="right") - 1
            for k in np.unique(which_u):
                curves, per_job = lst[k][1].result()
                rows = np.flatnonzero((rsrc >= 0) & (which_r == k))
                if len(rows) == R:  # every row from this piece: one gather straight into the output
                    np.take(curves, rsrc - lst[k][0], axis=0, out=out)
                else:
                    out[rows] = curves[rsrc[rows] - lst[k][0]]
                opj[rows] = per_job
                pj_u[got[which_u == k]] = per_job
        cached_r = np.flatnonzero(rsrc < 0)
        cache = self._tier_cache(tier, npts)
        if len(cached_r):
            at = cache.find(kv[inv[cached_r]])
            out[cached_r] = cache.curves[at]
            opj[cached_r] = cache.pj[at]
        # masks this batch solved first: their cost is this batch's, and they enter the run cache
        own = np.flatnonzero(src >= start)
        spent[bi] += float(pj_u[own].sum())
        if kv is not None and len(own):
            # the first request row of each own mask carries its curve
            first = np.empty(len(uniq), dtype=np.int64)
            first[inv[::-1]] = np.arange(R - 1, -1, -1)
            cache.add(kv[own], out[first[own]], pj_u[own])
        return out, opj

    def evaluate_masks(self, requests):
        """Dedup on (n, q, mask) against the run cache and within the batch; solve the new jobs of each
        (n, q) group in one GPU batch; results [(curve, per_job)] in request order (runner.py:206-244)."""
        order: dict = {}
        for idx, (n, q, mask, tid) in enumerate(requests):
            order.setdefault((n, q), []).append(idx)
        groups, rows_of = [], []
        for (n, q), idxs in order.items():
            nunits = self.supercell(n).nunits
            groups.append((n, q, words_from_keys([requests[i][2] for i in idxs], nunits)))
            rows_of.append(idxs)

        def ids(gi, new, inv):
            first = {}
            for r, u in enumerate(inv):
                first.setdefault(int(u), r)
            return [requests[rows_of[gi][first[int(u)]]][3] for u in new]

        res, hits, spent = self._evaluate_words(groups, ids)
        out = [None] * len(requests)
        for (cu, pj), idxs in zip(res, rows_of):
            for r, i in enumerate(idxs):
                out[i] = (cu[r], float(pj[r]))
        return out, hits, spent

    # -- level sampling --
    def draw_configs(self, supercell, p_vac: float, stream_level: int, count: int):
        words = sample_masks(supercell.nunits, p_vac, self.master_seed, stream_level, 0, count)
        return [DefectConfiguration.from_key(supercell, k) for k in keys_from_words(words)]

    def _level_batch(self, level: int, n: int, nsamples: int, p_vac: float, with_cv: bool, stream_level=None):
        """Masks of one level (parents, + restricted quarters) as a batch of the seam."""
        q = self.q_of(n)
        sc = self.supercell(n)
        stream = level if stream_level is None else stream_level
        # weak-scaling replica: rank r of `world` draws the replicates [r*M, (r+1)*M) of the stream (split
        # mode: every rank draws the whole level)
        rank, _ = self.shard
        m0 = rank * nsamples if self.shard_mode == "replicas" else 0
        if self.rng == "device":
            words, sub = self._draw_device(sc, p_vac, stream, m0, nsamples, with_cv)
        else:
            words = sample_masks(sc.nunits, p_vac, self.master_seed, stream, m0, nsamples)
            sub = restrict_words(words, self.quarters(sc)) if with_cv else None  # [M, 4, w]
        groups = [(n, q, words)]
        if with_cv:
            nsub = n // 2
            groups.append((nsub, self.q_of(nsub), sub.reshape(nsamples * 4, -1)))

        def ids(gi, new, inv):  # task ids (level, replicate, "Q" / "CVr") of the first row of each new mask
            rows = first_rows(inv)[new]
            if gi == 0:
                return [(level, m0 + int(r), "Q") for r in rows]
            return [(level, m0 + int(r) // 4, f"CV{int(r) % 4 + 1}") for r in rows]

        return groups, ids

    def _draw_device(self, sc, p_vac, stream_level, m0, count, with_cv):
        """Masks [count, w] (and quarter masks [count, 4, ws]) drawn on the GPU - the device port of the
        reference sampler (hx_sample_masks_device: SeedSequence -> PCG64 -> random() < p, bit-identical to
        disorder.py:66-81) and quarter restriction (hx_restrict_masks_device, disorder.py:84-94) - then copied
        to the host, where the run cache keys them (runner.py:213-233)."""
        import torch

        dev = torch.device("cuda", self.device)
        lib = _lib.load()
        st = _rng_stream(self.device)
        nunits = sc.nunits
        w = max(1, (nunits + 63) // 64)
        with torch.cuda.stream(st):
            d = torch.empty((max(count, 1), w), dtype=torch.int64, device=dev)
            _lib.check(lib.hx_sample_masks_device(self.master_seed, stream_level, m0, count, p_vac, nunits, d.data_ptr(),
                                                  st.cuda_stream), "hx_sample_masks_device")
            q = None
            if with_cv:
                part = self.quarters(sc)
                assign, umap = _quarter_maps(part, self.device)
                sub_units = part.subcells[0].nunits
                ws = max(1, (sub_units + 63) // 64)
                q = torch.empty((max(count, 1) * 4, ws), dtype=torch.int64, device=dev)
                _lib.check(lib.hx_restrict_masks_device(d.data_ptr(), count, nunits, assign.data_ptr(), umap.data_ptr(),
                                                        sub_units, q.data_ptr(), st.cuda_stream),
                           "hx_restrict_masks_device")
            words = d[:count].cpu().numpy().view(np.uint64)
            sub = None if q is None else q[:4 * count].cpu().numpy().view(np.uint64).reshape(count, 4, ws)
        return words, sub

    def _level_finish(self, level, n, nsamples, with_cv, evaluated):
        """Level terms + moments from the seam's results for the level's batch (runner.py:281-311)."""
        res, hits, spent = evaluated
        q = self.q_of(n)
        npts = self.grid.npoints
        full, pj = res[0]
        nominal = float(pj.sum())
        quarters = None
        if with_cv:
            qc, qpj = res[1]
            quarters = qc.reshape(nsamples, 4, npts)
            nominal += float(qpj.sum())
        # without the CV the level terms are the curves themselves: no device round trip for them
        terms, mean, var = level_moments(full, quarters, self.device, want_terms=quarters is not None)
        rank, world = self.shard
        if world > 1 and self.shard_mode == "replicas":
            # exact cross-rank combination (fixed-point limbs, int64 all-reduce): the bits of one process
            # drawing all world * M replicates
            import torch

            from ._dist import all_reduce

            dev = torch.device("cuda", self.device)
            mean, var = exact_level_moments(torch.as_tensor(full).to(dev),
                                            None if quarters is None else torch.as_tensor(quarters).to(dev),
                                            nsamples * world, allreduce=all_reduce)
            nsamples_all = nsamples * world
        else:
            nsamples_all = nsamples
        self.io_bytes[0] += full.nbytes + (0 if quarters is None else quarters.nbytes)
        self.io_bytes[1] += (0 if terms is None else full.nbytes) + 2 * mean.numel() * 8
        terms = full if terms is None else terms.cpu().numpy()  # no CV: terms is full itself (runner.py:297)
        cv = None
        if quarters is not None:
            # cv exactly as the reference forms it: ((q1 + q2) + q3 + q4) * 0.25
            cv = np.zeros((nsamples, npts))
            for r in range(4):
                cv += quarters[:, r, :]
            cv *= 0.25
        stats = LevelStats(level=level, n=n, q=q, nsamples=nsamples_all, mean=mean.cpu().numpy(),
                           sample_variance=var.cpu().numpy() if nsamples_all > 1 else None,
                           work_per_sample=nominal / nsamples, wall_seconds=spent, cache_hits=hits)
        return LevelSampleSet(stats=stats, terms=terms, full=full, cv=cv)

    def sample_level(self, level: int, n: int, nsamples: int, p_vac: float, with_cv: bool, stream_level=None):
        """Draw outcomes and evaluate the level terms with the quarter CV (runner.py:254-311)."""
        batch = self._level_batch(level, n, nsamples, p_vac, with_cv, stream_level)
        return self._level_finish(level, n, nsamples, with_cv, self._evaluate_batches([batch])[0])

    # -- mode drivers (runner.py:315-419) --
    def run_mc(self, plan: LevelPlan):
        level = plan.num_levels
        sset = self.sample_level(level, plan.ns[-1], plan.samples[-1], plan.p_vac, with_cv=False)
        return combine_levels(self.grid, [sset.stats], total_wall_seconds=sset.stats.wall_seconds), sset

    def run_mlmc(self, plan: LevelPlan):
        """All levels of the plan (runner.py:315-340).  The levels are deduplicated in order (the same
        cache hits as sampling them one after another) but their new masks are solved in one concurrent
        submission - every (n, q) tier of every level in flight at once."""
        levels = list(enumerate(zip(plan.ns, plan.samples), start=1))
        # drawn lazily: the largest tier's level first, so its solve starts while the others are drawn
        batches = [functools.partial(self._level_batch, idx, n, m, plan.p_vac, idx > 1) for idx, (n, m) in levels]
        tiers_of = [[(n, self.q_of(n))] + ([(n // 2, self.q_of(n // 2))] if idx > 1 else []) for idx, (n, _) in levels]
        sets = [None] * len(levels)

        def finish(bi, ev):  # each level's terms/moments as soon as its curves are in
            idx, (n, m) = levels[bi]
            sets[bi] = self._level_finish(idx, n, m, idx > 1, ev)

        self._evaluate_batches(batches, on_batch=finish, tiers_of=tiers_of)
        total = sum(s.stats.wall_seconds for s in sets)
        return combine_levels(self.grid, [s.stats for s in sets], total_wall_seconds=total), sets

    def run_slmc_reference(self, plan: LevelPlan, nsamples: int):
        level = plan.num_levels
        return self.sample_level(level, plan.ns[-1], nsamples, plan.p_vac, with_cv=False,
                                 stream_level=SLMC_STREAM_OFFSET + level)

    def run_rates(self, plan: LevelPlan, window=None) -> RatesResult:
        """Standalone per-level statistics (every level with its quarter CV) and the fitted exponents
        (runner.py:347-378): variance of Q_l, of the CV difference, the bias proxies |mean_l - mean_{l+1}| over
        the energy window and the per-sample cost.  The levels go to the seam as one concurrent submission,
        deduplicated in level order (the cache hits of sampling them one after another)."""
        mask = window_mask(self.grid, window)
        for n in plan.ns:
            if n % 2:
                raise ValueError("rate estimation needs even supercell factors for the CV")
        levels = list(enumerate(zip(plan.ns, plan.samples), start=1))
        batches = [functools.partial(self._level_batch, idx, n, m, plan.p_vac, True) for idx, (n, m) in levels]
        tiers_of = [[(n, self.q_of(n)), (n // 2, self.q_of(n // 2))] for _, (n, _) in levels]
        sets = [None] * len(levels)

        def finish(bi, ev):
            idx, (n, m) = levels[bi]
            sets[bi] = self._level_finish(idx, n, m, True, ev)

        self._evaluate_batches(batches, on_batch=finish, tiers_of=tiers_of)
        records, means = [], []
        for sset in sets:
            _, var_q = mean_and_variance(sset.full)
            mean_q = np.mean(sset.full, axis=0)
            means.append(mean_q)
            records.append({"set": sset, "n": sset.stats.n, "variance_q": float(np.mean(var_q[mask])),
                            "variance_diff": float(np.mean(sset.stats.sample_variance[mask])),
                            "seconds_per_sample": sset.stats.work_per_sample})
        proxies = [float(np.mean(np.abs(means[i] - means[i + 1])[mask])) for i in range(len(means) - 1)]
        rates = fit_rates(plan.ns, bias_proxies=proxies if len(proxies) >= 2 else None,
                          variances=[r["variance_q"] for r in records],
                          cv_diff_variances=[r["variance_diff"] for r in records],
                          work=[r["seconds_per_sample"] for r in records])
        return RatesResult(records=records, rates=rates, bias_proxies=proxies)

    def band_structure(self, n: int, bz_mode: str | None = None):
        """Unperturbed bands of the nu = n supercell on its (n, q) grid - the CLI's "bands" mode
        (cli.py:132-152: solve_bands(model, supercell, None, make_bz_grid(..., bz_mode)))."""
        grid = make_bz_grid(self.model.lattice_spec(), n, self.q_of(n), bz_mode or self.bz_mode)
        return solve_bands(self.model, self.supercell(n), None, grid, cell=self.cell(n))

    def run_exhaustive(self, n: int, p_vac: float, symmetry_reduce: bool = False, cap: int = 24):
        """Exact expectation over all 2^N outcomes with binomial weights (runner.py:380-415)."""
        if symmetry_reduce:
            raise NotImplementedError("translation-orbit reduction is outside the GPU hot path")
        sc = self.supercell(n)
        q = self.q_of(n)
        pairs = list(enumerate_configs(sc, p_vac, cap=cap))
        weight_sum = math.fsum(w for _, w in pairs)
        if abs(weight_sum - 1.0) > 1e-12:
            raise ArithmeticError(f"enumeration weights sum to {weight_sum!r}, not 1")
        masks = [c.key for c, _ in pairs]
        results, hits, spent = self.evaluate_masks([(n, q, m, ("exhaustive", m)) for m in masks])
        m1 = np.zeros(self.grid.npoints)
        m2 = np.zeros(self.grid.npoints)
        for (_, w), (c, _) in zip(pairs, results):
            m1 += w * c
            m2 += w * c * c
        return ExhaustiveResult(mean=m1, variance=np.maximum(m2 - m1 * m1, 0.0), weight_sum=weight_sum,
                                nconfigs=len(pairs), evaluations=len(masks) - hits, cache_hits=hits,
                                wall_seconds=spent, n=n, q=q)

    def unperturbed_curve(self, n: int) -> np.ndarray:
        results, _, _ = self.evaluate_masks([(n, self.q_of(n), 0, ("unperturbed", n))])
        return results[0][0]
