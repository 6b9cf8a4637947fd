"""Brillouin-zone grids and per-sample band solves on the GPU (spectrum.py:37-145).

`solve_bands` runs the same fused device pipeline as the batch path (assembly -> Householder
tridiagonalisation -> Sturm bisection) for one sample and returns the ascending eigenvalues per
k-point.  Eigensolver failures come back as per-k status codes and are raised as SolverError with
the reference's message text (spectrum.py:109-117).
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .models import CompiledCell, compile_cell

__all__ = ["BzGrid", "BandGrid", "SolverError", "make_bz_grid", "solve_bands", "estimate_solve_cost", "eval_batch",
           "time_reversal_reduce", "use_time_reversal"]


class SolverError(RuntimeError):
    """Eigensolver failure, tagged with the offending k-point."""


@dataclass(frozen=True, eq=False)
class BzGrid:
    n: int
    q: int
    mode: str
    kpoints: np.ndarray = field(repr=False)
    weights: np.ndarray = field(repr=False)

    @property
    def nk(self) -> int:
        return len(self.weights)


def _rotation(angle):
    c, s = np.cos(angle), np.sin(angle)
    return np.array([[c, -s], [s, c]])


def make_bz_grid(spec, n: int, q: int, mode: str = "full") -> BzGrid:
    """q x q corner grid on the supercell BZ rhombus; 'full' appends the +-120 deg copies (spectrum.py:59-84)."""
    if q < 1:
        raise ValueError(f"q must be >= 1, got {q}")
    if n < 1:
        raise ValueError(f"supercell factor must be >= 1, got {n}")
    if mode not in ("reduced", "full"):
        raise ValueError(f"unknown BZ mode {mode!r}")
    b1, b2 = spec.reciprocal_vectors()
    ii, jj = np.meshgrid(np.arange(q), np.arange(q), indexing="ij")
    base = ii.reshape(-1, 1) * (b1 / (n * q))[None, :] + jj.reshape(-1, 1) * (b2 / (n * q))[None, :]
    if mode == "full":
        kp = np.concatenate([base, base @ _rotation(2.0 * np.pi / 3.0).T, base @ _rotation(4.0 * np.pi / 3.0).T])
    else:
        kp = base
    return BzGrid(n=n, q=q, mode=mode, kpoints=kp, weights=np.full(len(kp), 1.0 / len(kp)))


def use_time_reversal() -> bool:
    """k -> -k pairing of the IDOS batches (HX_NO_TIME_REVERSAL=1 disables it)."""
    return os.environ.get("HX_NO_TIME_REVERSAL", "0") in ("", "0")


def time_reversal_reduce(spec, n: int, kpoints: np.ndarray):
    """Representatives and multiplicities of `kpoints` under k -> -k modulo the supercell reciprocal
    lattice (b1/n, b2/n).  For real-amplitude models H(-k) = conj(H(k)) (and S likewise), so both have the
    spectrum of H(k): the IDOS sum over the reference's grid (weights 1/nk, spectrum.py:59-84) equals the
    sum over the representatives with weights mult/nk.  On the q x q corner grid the pairs are
    (i, j) <-> (-i mod q, -j mod q); the time-reversal-invariant points keep multiplicity 1."""
    kp = np.asarray(kpoints, dtype=np.float64).reshape(-1, 2)
    b1, b2 = spec.reciprocal_vectors()
    B = np.stack([np.asarray(b1) / n, np.asarray(b2) / n], axis=1)
    frac = np.linalg.solve(B, kp.T).T

    def key(f):
        r = np.round(np.mod(f, 1.0), 9)
        return tuple(np.mod(r, 1.0))

    index = {}  # key of a representative -> its slot
    reps, mult = [], []
    for i, f in enumerate(frac):
        j = index.get(key(-f))
        if j is not None and mult[j] == 1:  # the partner of an earlier, still unpaired point
            mult[j] = 2
            continue
        index.setdefault(key(f), len(reps))
        reps.append(i)
        mult.append(1)
    return np.ascontiguousarray(kp[reps]), np.asarray(mult, dtype=np.int32)


@dataclass(frozen=True, eq=False)
class BandGrid:
    grid: BzGrid
    energies: np.ndarray = field(repr=False)
    solve_seconds: float = 0.0

    @property
    def nbands(self) -> int:
        return self.energies.shape[1]


def _egrid(lo, step, npts, delta):
    g = _lib.EGrid()
    g.e0, g.step, g.npts, g.delta = float(lo), float(step), int(npts), float(delta)
    return g


def raise_status(status: np.ndarray, kpoints: np.ndarray, what: str = "eigensolver"):
    """Map HX_ST_* codes to the reference's SolverError messages (spectrum.py:109-117)."""
    bad = np.argwhere((status == _lib.HX_ST_NOT_PD) | (status == _lib.HX_ST_NONFINITE))
    if len(bad) == 0:
        return
    row = tuple(bad[0])
    k = kpoints[row[-1]]
    if status[row] == _lib.HX_ST_NOT_PD:
        raise SolverError(f"overlap matrix not positive definite at k=({k[0]:.6g}, {k[1]:.6g})")
    raise SolverError(f"eigensolver failed at k=({k[0]:.6g}, {k[1]:.6g}): non-finite value")


def eval_batch(cell: CompiledCell, kpoints: np.ndarray, words: np.ndarray, lo: float, step: float, npts: int,
               delta: float, want_eigs: bool = False, sharp: bool = False, ctx=None, kmult=None):
    """Host-buffer call of hx_eval_idos_batch for one (n, q) group: curves [M, npts] (+ eigs, status).
    ctx: the hx context to use (default: the device's primary context); the call blocks until done and
    releases the GIL, so groups on different contexts run concurrently from different threads."""
    lib = _lib.load()
    if ctx is None:
        ctx = _lib.Device.ctx(cell.device)
    words = np.ascontiguousarray(words, dtype=np.uint64)
    M = words.shape[0]
    kp = np.ascontiguousarray(kpoints, dtype=np.float64).reshape(-1, 2)
    nk = kp.shape[0]
    curves = np.zeros((M, npts))
    status = np.zeros((M, nk), dtype=np.int32)
    eigs = np.empty((M, nk, cell.dim)) if want_eigs else None
    g = _egrid(lo, step, npts, delta)
    if kmult is not None:
        # k-point multiplicities (time-reversal pairs): smoothed IDOS only
        if want_eigs or sharp:
            raise ValueError("k-point multiplicities apply to the smoothed IDOS without eigenvalue output")
        km = np.ascontiguousarray(kmult, dtype=np.int32)
        if km.shape != (nk,):
            raise ValueError("one multiplicity per k-point")
        _lib.check(lib.hx_eval_idos_batch_k(ctx, cell.handle, _lib.ptr(kp), _lib.ptr(km), nk, _lib.ptr(words), M,
                                            C.byref(g), _lib.ptr(curves), _lib.ptr(status)), "hx_eval_idos_batch_k")
        return curves, None, status
    fn = lib.hx_eval_sharp_batch if sharp else lib.hx_eval_idos_batch
    _lib.check(fn(ctx, cell.handle, _lib.ptr(kp), nk, _lib.ptr(words), M, C.byref(g), _lib.ptr(curves),
                  _lib.ptr(eigs) if want_eigs else 0, _lib.ptr(status)), "hx_eval_idos_batch")
    return curves, eigs, status


def solve_bands(model, supercell, defects, grid: BzGrid, cell: CompiledCell | None = None) -> BandGrid:
    """Ascending (generalized) eigenvalues for every grid point of one sample (spectrum.py:120-134)."""
    if cell is None:
        cell = compile_cell(model, supercell)
    vacant = () if defects is None else defects.vacant
    keep = cell.configure(vacant)
    d = int(keep.sum())
    words = cell.mask_words(vacant).reshape(1, -1)
    t0 = time.perf_counter()
    _, eigs, status = eval_batch(cell, grid.kpoints, words, 0.0, 1.0, 1, 1.0, want_eigs=True)
    raise_status(status, grid.kpoints)
    return BandGrid(grid=grid, energies=np.ascontiguousarray(eigs[0, :, :d]),
                    solve_seconds=time.perf_counter() - t0)


def estimate_solve_cost(n: int, q: int, orbitals_per_cell: int, mode: str = "full", unit_cost: float = 1.0) -> float:
    """Work model (n^2 orbitals)^3 per k-point x k-point count (spectrum.py:137-145)."""
    nk = q * q * (3 if mode == "full" else 1)
    return unit_cost * nk * float(n * n * orbitals_per_cell) ** 3
