"""Device-resident MLMC level pipeline (no host round trips): the throughput path used by bench.py.

Per level: vacancy masks (device RNG, bit-exact with the reference sampler) -> quarter restriction
(device) -> in-level dedup of (n, q, mask) keys (sort-unique on the device, the reference's
evaluate_masks semantics within the level) -> one hx_eval_idos_batch_device per (n, q) tier ->
gather per-request curves -> CV terms + moments (hx_level_moments_device).  Multi-rank: samples of
each level are sharded contiguously across ranks; per-rank sums (sum term, sum term^2) are combined
with one all-reduce per level (runner.py:281-299 + mlmc.py:143-154 semantics for the mean).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .geometry import build_supercell, partition_quarters
from .models import compile_cell
from .solver import make_bz_grid, time_reversal_reduce, use_time_reversal


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
                 device: int = 0):
        self.model = model
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

        Weak scaling: every rank processes a full level of M samples from its own replicate range."""
        m0 = rank * M_total
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

    def _eval(self, n, words: torch.Tensor):
        """Dedup rows, solve unique masks, return per-row curves [rows, npts] (device)."""
        uniq, inv = torch.unique(words, dim=0, return_inverse=True)
        return self._solve(n, uniq.contiguous(), self.ctx, self.stream)[0][inv]

    def _solve(self, n, uniq: torch.Tensor, ctx, stream):
        """Curves [U, npts] of the unique masks `uniq`, enqueued on `stream` with context `ctx`.  The
        outputs (curves, status) are allocated on the caller's current stream, which must wait on `stream`
        before using or releasing them."""
        cell = self.cell(n)
        q = self.q_of(n)
        kp, kmult = self.kpoints(n, q)
        U = uniq.shape[0]
        curves = torch.empty((U, self.npts), dtype=torch.float64, device=self.dev)
        status = torch.empty((U, kp.shape[0]), dtype=torch.int32, device=self.dev)
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
        return curves, status

    def run_level(self, inp: LevelInputs):
        """Returns device tensors (sum term [npts], sum term^2 [npts]) for this rank's shard."""
        npts = self.npts
        sums = torch.zeros(2 * npts, dtype=torch.float64, device=self.dev)
        if inp.M == 0:
            return sums
        full = self._eval(inp.n, inp.parent)
        quarters = None
        if inp.with_cv:
            quarters = self._eval(inp.n // 2, inp.quarters).reshape(inp.M, 4, npts)
        _lib.check(self.lib.hx_level_moments_device(full.data_ptr(), 0 if quarters is None else quarters.data_ptr(),
                                                    inp.M, npts, 0, 0, 0, sums.data_ptr(), self.stream.cuda_stream),
                   "hx_level_moments_device")
        return sums


    def run_levels(self, inputs):
        """All levels at once: every (level, fine / coarse) solve on its own stream and context, so the
        latency-bound tails of one tier (e.g. the nu = 32 bulge chase on 64 matrices) overlap with the
        others.  Same results as run_level per input (each solve is deterministic); returns the list of
        per-level sums on the current stream."""
        main = self.stream
        jobs = []  # (input index, n, uniq, inv)
        for i, inp in enumerate(inputs):
            if inp.M == 0:
                continue
            u, inv = torch.unique(inp.parent, dim=0, return_inverse=True)
            jobs.append((i, inp.n, u.contiguous(), inv))
            if inp.with_cv:
                u, inv = torch.unique(inp.quarters, dim=0, return_inverse=True)
                jobs.append((i, inp.n // 2, u.contiguous(), inv))
        start = torch.cuda.Event()
        start.record(main)
        outs = [None] * len(jobs)
        # largest tier first (lane 0 = high priority)
        order = sorted(range(len(jobs)), key=lambda j: -self.cell(jobs[j][1]).dim)
        for lane, j in enumerate(order):
            i, n, uniq, inv = jobs[j]
            ctx, stream = self._lane(lane)
            stream.wait_event(start)
            curves, status = self._solve(n, uniq, ctx, stream)
            done = torch.cuda.Event()
            done.record(stream)
            outs[j] = (curves, done, status)
        res = []
        k = 0
        for inp in inputs:
            sums = torch.zeros(2 * self.npts, dtype=torch.float64, device=self.dev)
            if inp.M == 0:
                res.append(sums)
                continue
            curves, done, _ = outs[k]
            main.wait_event(done)
            full = curves[jobs[k][3]]
            k += 1
            quarters = None
            if inp.with_cv:
                curves, done, _ = outs[k]
                main.wait_event(done)
                quarters = curves[jobs[k][3]].reshape(inp.M, 4, self.npts)
                k += 1
            _lib.check(self.lib.hx_level_moments_device(full.data_ptr(),
                                                        0 if quarters is None else quarters.data_ptr(), inp.M,
                                                        self.npts, 0, 0, 0, sums.data_ptr(), main.cuda_stream),
                       "hx_level_moments_device")
            res.append(sums)
        for _, done, _ in outs:  # every lane joins the main stream before its outputs can be released
            main.wait_event(done)
        return res


def kept_dims(cell, uniq_words: torch.Tensor) -> np.ndarray:
    """Kept dimension d of each unique mask (for the algorithmic 16/3 d^3 FLOP count)."""
    w = uniq_words.cpu().numpy().view(np.uint64)
    nunits = cell.supercell.nunits
    bits = np.unpackbits(w.view(np.uint8), axis=1, bitorder="little")[:, :nunits].astype(bool)
    per_unit = np.array([len(d) for d in cell.unit_dofs], dtype=np.int64)
    removed = bits.astype(np.int64) @ per_unit if nunits else np.zeros(len(w), np.int64)
    return cell.dim - removed
