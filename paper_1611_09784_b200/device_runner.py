"""Device-resident MLMC level pipeline (no host round trips): the throughput path used by bench.py.

Per level: vacancy masks (device RNG, bit-exact with the reference sampler, disorder.py:57-81) -> quarter
restriction (device, disorder.py:84-94) -> dedup of (n, q, mask) keys within the level (sort-unique on the
device: the reference's evaluate_masks semantics within the level, runner.py:206-244) -> one
hx_eval_idos_batch_device per (n, q) tier -> gather per-request curves -> CV terms + EXACT level moments
(fixed-point sums, hx_level_sums_fixed_device; runner.py:281-299, mlmc.py:143-154).

Multi-rank, two modes:
  replicas (weak scaling, bench default): rank r draws the replicates [r*M, (r+1)*M) of every level stream;
     the fixed-point limbs of the level sums are all-reduced (int64), so the level mean / variance are the
     bits of one device running all world*M replicates.
  split (strong scaling): every rank draws the whole level (cheap), dedups it identically, solves a
     contiguous slice of the unique masks balanced by sum d^3 (d = kept dimension), and the slices' curves
     are all-gathered; the moments are then the bits of the single-device run (and cache semantics are the
     single-device ones).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .geometry import build_supercell, partition_quarters
from .models import compile_cell
from .estimators import exact_level_moments
from .solver import make_bz_grid, time_reversal_reduce, use_time_reversal

_MERGE_TIERS = __import__("os").environ.get("HX_MERGE_TIERS", "0") == "1"
_LANES = int(__import__("os").environ.get("HX_LANES", "3"))
_JOINT_DEDUP = __import__("os").environ.get("HX_JOINT_DEDUP", "1") != "0"
# HX_SUBMIT_THREADS=1: every lane's tier solves are enqueued from the lane's own submission thread
_SUBMIT_THREADS = __import__("os").environ.get("HX_SUBMIT_THREADS", "1") != "0"


class _Done:
    """Future-like wrapper of an already available result."""

    def __init__(self, value):
        self._value = value

    def result(self):
        return self._value
_LANE_MAP = [int(x) for x in __import__("os").environ.get("HX_LANE_MAP", "").split(",") if x]


@dataclass
class LevelInputs:
    level: int
    n: int
    q: int
    M: int            # samples on this rank
    m0: int           # first replicate index of this rank
    with_cv: bool
    parent: torch.Tensor          # [M, w] int64 view of uint64 words
    quarters: torch.Tensor | None  # [M*4, ws]


class DeviceMlmc:
    def __init__(self, model, nq: int, delta: float, master_seed: int, lo: float, hi: float, npts: int,
                 device: int = 0, group=None, mode: str = "replicas"):
        if mode not in ("replicas", "split"):
            raise ValueError(f"unknown multi-rank mode {mode!r}")
        self.model = model
        self.mode = mode
        self.group = group  # torch.distributed process group (None: single rank)
        self.statuses = []  # per-solve status tensors of the last run (check_status)
        self.nq = nq
        self.delta = delta
        self.seed = master_seed
        self.lo, self.hi, self.npts = lo, hi, npts
        self.step = (hi - lo) / (npts - 1)
        self.device = device
        self.dev = torch.device("cuda", device)
        self.lib = _lib.load()
        self.ctx = _lib.Device.ctx(device)
        self._cells = {}
        self._parts = {}
        self._kpts = {}
        self.stream = torch.cuda.current_stream(self.dev)
        # per-call accounting for the roofline: list of (n, nmats, flops, event pair)
        self.records = []
        self.record = False
        self._lanes = []  # (ctx, stream) pairs for run_levels

    def _lane(self, i):
        # lane 0 carries the largest tier (the critical path of a level set) on a high-priority stream, so
        # its latency-bound kernels (e.g. the bulge chase on a few large matrices) are not starved of SMs
        # by the throughput-bound tiers running beside it
        while len(self._lanes) <= i:
            prio = -1 if not self._lanes else 0
            self._lanes.append((_lib.Device.new_ctx(self.device), torch.cuda.Stream(self.dev, priority=prio)))
        return self._lanes[i]

    def _submitter(self, lane):
        from concurrent.futures import ThreadPoolExecutor

        if not hasattr(self, "_submitters"):
            self._submitters = {}
        if lane not in self._submitters:
            self._submitters[lane] = ThreadPoolExecutor(max_workers=1, thread_name_prefix=f"hx-lane{lane}")
        return self._submitters[lane]

    def cell(self, n):
        if n not in self._cells:
            self._cells[n] = compile_cell(self.model, build_supercell(self.model.lattice_spec(), n), self.device)
        return self._cells[n]

    def part(self, n):
        if n not in self._parts:
            p = partition_quarters(self._cells[n].supercell if n in self._cells else
                                   build_supercell(self.model.lattice_spec(), n))
            self._parts[n] = (p, torch.from_numpy(p.unit_assignment.astype(np.int32)).to(self.dev),
                              torch.from_numpy(p.unit_map.astype(np.int32)).to(self.dev))
        return self._parts[n]

    def q_of(self, n):
        return self.nq // n

    def kpoints(self, n, q):
        """(k-points, multiplicities): the reduced grid, time-reversal pairs merged for real-amplitude
        models (solver.time_reversal_reduce; multiplicities None otherwise)."""
        key = (n, q)
        if key not in self._kpts:
            kp = np.ascontiguousarray(make_bz_grid(self.model.lattice_spec(), n, q, "reduced").kpoints)
            if use_time_reversal() and self.cell(n).time_reversal_symmetric:
                self._kpts[key] = time_reversal_reduce(self.model.lattice_spec(), n, kp)
            else:
                self._kpts[key] = (kp, None)
        return self._kpts[key]

    def prepare(self, level, n, M_total, p, with_cv, rank=0, world=1) -> LevelInputs:
        """Masks for this rank's replicates [rank*M, (rank+1)*M) (device RNG) + quarter masks.

        replicas: every rank processes a full level of M samples from its own replicate range (weak scaling).
        split: every rank draws the whole level [0, M); the unique masks are split in run_levels."""
        m0 = rank * M_total if self.mode == "replicas" else 0
        M = M_total
        cell = self.cell(n)
        nunits = cell.supercell.nunits
        w = max(1, (nunits + 63) // 64)
        parent = torch.zeros((max(M, 1), w), dtype=torch.int64, device=self.dev)
        st = self.stream.cuda_stream
        _lib.check(self.lib.hx_sample_masks_device(self.seed, level, m0, M, p, nunits, parent.data_ptr(), st),
                   "hx_sample_masks_device")
        quarters = None
        if with_cv:
            part, assign, umap = self.part(n)
            sub_units = part.subcells[0].nunits
            ws = max(1, (sub_units + 63) // 64)
            quarters = torch.zeros((max(M, 1) * 4, ws), dtype=torch.int64, device=self.dev)
            _lib.check(self.lib.hx_restrict_masks_device(parent.data_ptr(), M, nunits, assign.data_ptr(),
                                                         umap.data_ptr(), sub_units, quarters.data_ptr(), st),
                       "hx_restrict_masks_device")
        return LevelInputs(level, n, self.q_of(n), M, m0, with_cv, parent[:M], None if quarters is None else
                           quarters[:4 * M])

    def _solve(self, n, uniq: torch.Tensor, ctx, stream):
        """Curves [U, npts] of the unique masks `uniq`, enqueued on `stream` with context `ctx`.  The
        outputs (curves, status) are allocated on the caller's current stream, which must wait on `stream`
        before using or releasing them."""
        curves, status = self._solve_alloc(n, uniq)
        self._solve_launch(n, uniq, curves, status, ctx, stream)
        return curves, status

    def _solve_alloc(self, n, uniq: torch.Tensor):
        """Output buffers of one tier solve, allocated on the caller's current stream."""
        kp, _ = self.kpoints(n, self.q_of(n))
        U = uniq.shape[0]
        return (torch.empty((U, self.npts), dtype=torch.float64, device=self.dev),
                torch.empty((U, kp.shape[0]), dtype=torch.int32, device=self.dev))

    def _solve_launch(self, n, uniq, curves, status, ctx, stream, after=None):
        """Enqueue the solve on `stream` (after the event `after`); may run on a lane's submission thread: the C
        call releases the GIL, so the caller goes on deduplicating the next tier while this one is enqueued."""
        torch.cuda.set_device(self.dev)  # a submission thread starts on device 0
        if after is not None:
            stream.wait_event(after)
        cell = self.cell(n)
        q = self.q_of(n)
        kp, kmult = self.kpoints(n, q)
        U = uniq.shape[0]
        g = _lib.EGrid()
        g.e0, g.step, g.npts, g.delta = self.lo, self.step, self.npts, self.delta
        ev = None
        if self.record:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(stream)
        if kmult is None:
            _lib.check(self.lib.hx_eval_idos_batch_device(ctx, cell.handle, _lib.ptr(kp), kp.shape[0],
                                                          uniq.data_ptr(), U, C.byref(g), curves.data_ptr(), 0,
                                                          status.data_ptr(), stream.cuda_stream),
                       "hx_eval_idos_batch_device")
        else:
            _lib.check(self.lib.hx_eval_idos_batch_device_k(ctx, cell.handle, _lib.ptr(kp), _lib.ptr(kmult),
                                                            kp.shape[0], uniq.data_ptr(), U, C.byref(g),
                                                            curves.data_ptr(), status.data_ptr(),
                                                            stream.cuda_stream),
                       "hx_eval_idos_batch_device_k")
        if self.record:
            ev[1].record(stream)
            self.records.append({"n": n, "N": cell.dim, "unique": U, "nk": kp.shape[0], "events": ev,
                                 "uniq": uniq, "cell": cell})
        done = torch.cuda.Event()
        done.record(stream)
        return done

    def _world(self):
        if self.group is None:
            return 0, 1
        import torch.distributed as dist

        return dist.get_rank(self.group), dist.get_world_size(self.group)

    def _allreduce(self):
        if self.group is None or self.mode != "replicas":
            return None
        from ._dist import all_reduce

        return lambda t: all_reduce(t, group=self.group)

    def _split(self, n, uniq):
        """split mode: [start, stop) of this rank's contiguous slice of the unique masks, balanced by d^3, and
        the cut points of every rank (all ranks compute the same cuts)."""
        rank, world = self._world()
        U = uniq.shape[0]
        if world == 1 or U == 0:
            return 0, U, [0, U]
        d = kept_dims_device(self.cell(n), uniq).to(torch.float64)
        c = torch.cumsum(d * d * d, 0)
        targets = c[-1] * torch.arange(1, world, dtype=torch.float64, device=self.dev) / world
        cuts = [0] + torch.searchsorted(c, targets).add_(1).clamp_(max=U).tolist() + [U]
        for i in range(1, len(cuts)):
            cuts[i] = max(cuts[i], cuts[i - 1])
        return cuts[rank], cuts[rank + 1], cuts

    def _gather(self, curves, cuts):
        """split mode: all ranks' slices of the unique curves, in unique order."""
        rank, world = self._world()
        if world == 1:
            return curves
        width = max(b - a for a, b in zip(cuts[:-1], cuts[1:]))
        pad = torch.zeros((width, self.npts), dtype=torch.float64, device=self.dev)
        pad[: curves.shape[0]] = curves
        out = torch.empty((world * width, self.npts), dtype=torch.float64, device=self.dev)
        from ._dist import all_gather_into_tensor

        all_gather_into_tensor(out, pad, group=self.group)
        return torch.cat([out[r * width: r * width + (cuts[r + 1] - cuts[r])] for r in range(world)])

    def run_level(self, inp: LevelInputs):
        """(mean [npts], var [npts]) device tensors of one level, tiers one after another on the main stream."""
        return self.run_levels([inp], concurrent=False)[0]

    def run_levels(self, inputs, concurrent: bool = True):
        """All levels at once: every (level, fine / coarse) solve on its own stream and context, so the
        latency-bound tails of one tier (e.g. the nu = 32 bulge chase on 64 matrices) overlap with the
        others.  Each solve is deterministic, so the results do not depend on the schedule.  Returns the
        per-level (mean, var) on the current stream (exact fixed-point moments, combined over the ranks)."""
        main = self.stream
        # (input index, n, words) of every (level, tier) solve
        specs = []
        for i, inp in enumerate(inputs):
            if inp.M == 0:
                continue
            for n, words in ((inp.n, inp.parent), (inp.n // 2, inp.quarters)):
                if words is not None:
                    specs.append((i, n, words))

        def dedup(n, words):
            u, inv = torch.unique(words, dim=0, return_inverse=True)
            a, b, cuts = (0, u.shape[0], None) if self.mode == "replicas" else self._split(n, u)
            return u[a:b].contiguous(), inv, cuts

        jobs = [None] * len(specs)  # (input index, n, uniq slice of this rank, inv, cuts)
        outs = [None] * len(specs)
        self.statuses = []
        # largest tier first (lane 0 = high priority)
        by_size = sorted(range(len(specs)), key=lambda j: -self.cell(specs[j][1]).dim)
        if not _MERGE_TIERS:
            # every tier is deduplicated (main stream) and submitted (its lane) in turn, largest first: the largest
            # tier is on the GPU after its own torch.unique instead of after all of them (~1 ms of a c2 step)
            # Tiers of the same small cell (one-word masks: nu = 4 in c2, where a level's quarter masks repeat the
            # parent masks of the level below) are deduplicated TOGETHER and solved once - the cross-level hits of
            # the reference's run cache (runner.py:213-233; Engine.evaluate_masks does the same on the host).
            # HX_JOINT_DEDUP=0: every tier on its own.
            groups, seen = [], set()
            for j in by_size:
                if j in seen:
                    continue
                n = specs[j][1]
                same = [j2 for j2 in by_size if j2 not in seen and specs[j2][1] == n] \
                    if _JOINT_DEDUP and self.cell(n).supercell.nunits <= 64 else [j]
                seen.update(same)
                groups.append(same)
            for lane, js in enumerate(groups):
                j = js[0]
                i, n, _ = specs[j]
                words = specs[j][2] if len(js) == 1 else torch.cat([specs[j2][2] for j2 in js])
                uniq, inv, cuts = dedup(n, words)
                off = 0
                for j2 in js:
                    rows = specs[j2][2].shape[0]
                    jobs[j2] = (specs[j2][0], n, uniq, inv[off: off + rows], cuts)
                    off += rows
                ready = torch.cuda.Event()
                ready.record(main)
                # HX_LANES = L > 1 (default 3): the largest tier keeps lane 0, the others share lanes 1 .. L-1
                # round-robin (tiers on one lane run one after another); 0: one lane per tier.  Measured on c2
                # (7 tiers): 7 lanes 41.5 ms, 3 lanes 40.5 ms, 2 lanes 43.0 ms - the throughput-bound small tiers
                # gain nothing from running beside each other, and fewer co-resident kernels leave more L2 /
                # issue slots per kernel
                if _LANE_MAP:
                    lane = _LANE_MAP[min(lane, len(_LANE_MAP) - 1)]
                elif _LANES > 1 and lane > 0:
                    lane = 1 + (lane - 1) % (_LANES - 1)
                ctx, stream = self._lane(lane) if concurrent else (self.ctx, main)
                curves, status = self._solve_alloc(n, uniq)
                if concurrent and _SUBMIT_THREADS:
                    # one submission thread per lane (tiers of a lane stay in order; one host thread per context)
                    fut = self._submitter(lane).submit(self._solve_launch, n, uniq, curves, status, ctx, stream, ready)
                else:
                    fut = _Done(self._solve_launch(n, uniq, curves, status, ctx, stream, ready))
                for j2 in js:
                    outs[j2] = (curves, fut)
                self.statuses.append(status)
            outs = [None if o is None else (o[0], o[1].result()) for o in outs]  # enqueued: the `done` events
        else:
            # HX_MERGE_TIERS=1: the jobs of one tier (the same n) from different levels go to ONE batch call
            # (curves are batch independent, so only the packing of the GPU changes)
            for j, (i, n, words) in enumerate(specs):
                jobs[j] = (i, n) + dedup(n, words)
            start = torch.cuda.Event()
            start.record(main)
            groups = {}
            for j, (_, n, _, _, _) in enumerate(jobs):
                groups.setdefault(n, []).append(j)
            order = sorted(groups, key=lambda key: -self.cell(key).dim)
            for lane, key in enumerate(order):
                js = groups[key]
                n = jobs[js[0]][1]
                uniq = jobs[js[0]][2] if len(js) == 1 else torch.cat([jobs[j][2] for j in js]).contiguous()
                ctx, stream = self._lane(lane) if concurrent else (self.ctx, main)
                stream.wait_event(start)
                curves, status = self._solve(n, uniq, ctx, stream)
                done = torch.cuda.Event()
                done.record(stream)
                off = 0
                for j in js:
                    cnt = jobs[j][2].shape[0]
                    outs[j] = (curves[off: off + cnt], done)
                    off += cnt
                self.statuses.append(status)
        for _, done in outs:  # every lane joins the main stream before its outputs are used or released
            main.wait_event(done)
        allreduce = self._allreduce()
        res = []
        k = 0
        for inp in inputs:
            if inp.M == 0:
                z = torch.zeros(self.npts, dtype=torch.float64, device=self.dev)
                res.append((z, torch.full_like(z, float("nan"))))
                continue
            parts = []
            for _ in range(2 if inp.with_cv else 1):
                curves = outs[k][0]
                if jobs[k][4] is not None:
                    curves = self._gather(curves, jobs[k][4])
                parts.append(curves[jobs[k][3]])
                k += 1
            full = parts[0]
            quarters = parts[1].reshape(inp.M, 4, self.npts) if inp.with_cv else None
            _, world = self._world()
            m_total = inp.M * world if self.mode == "replicas" else inp.M
            res.append(exact_level_moments(full, quarters, m_total, allreduce))
        return res

    def check_status(self):
        """Raise if any (mask, k) solve of the last run reported a failure (HX_ST_NOT_PD / NONFINITE); the
        all-vacant HX_ST_EMPTY is a valid zero curve (runner.py:122-125)."""
        for st in self.statuses:
            bad = ((st != _lib.HX_ST_OK) & (st != _lib.HX_ST_EMPTY)).sum().item()
            if bad:
                raise RuntimeError(f"{bad} (mask, k) solves failed in the device pipeline")


def kept_dims_device(cell, uniq_words: torch.Tensor) -> torch.Tensor:
    """Kept dimension d of each mask row, on the device (int64 [rows])."""
    nunits = cell.supercell.nunits
    w = uniq_words.shape[1]
    shifts = torch.arange(64, dtype=torch.int64, device=uniq_words.device)
    bits = ((uniq_words.unsqueeze(-1) >> shifts) & 1).reshape(uniq_words.shape[0], 64 * w)[:, :nunits]
    per_unit = torch.tensor([len(d) for d in cell.unit_dofs], dtype=torch.int64, device=uniq_words.device)
    return cell.dim - (bits * per_unit).sum(1)


def kept_dims(cell, uniq_words: torch.Tensor) -> np.ndarray:
    """Kept dimension d of each unique mask (for the algorithmic 16/3 d^3 FLOP count)."""
    w = uniq_words.cpu().numpy().view(np.uint64)
    nunits = cell.supercell.nunits
    bits = np.unpackbits(w.view(np.uint8), axis=1, bitorder="little")[:, :nunits].astype(bool)
    per_unit = np.array([len(d) for d in cell.unit_dofs], dtype=np.int64)
    removed = bits.astype(np.int64) @ per_unit if nunits else np.zeros(len(w), np.int64)
    return cell.dim - removed
