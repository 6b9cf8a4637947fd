"""MC / MLMC estimator bookkeeping (mlmc.py:49-196).

Per-level moments are formed on the GPU by `level_moments` (hx_level_moments_device): the control-
variate term full - 0.25 * sum_r quarter_r, then the mean and the unbiased variance in fixed sample
order, reproducing np.mean / np.var(ddof=1) over axis 0 (mlmc.py:143-154) and the CV assembly
order of runner.py:281-299.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = ["LevelPlan", "LevelStats", "MlmcEstimate", "mean_and_variance", "level_moments", "exact_level_moments", "combine_levels",
           "control_variate_sample", "window_mask", "RateFit", "RateEstimates", "fit_loglog_slope", "fit_rates"]


@dataclass(frozen=True)
class LevelPlan:
    """Supercell factors doubling per level with n*q held constant (mlmc.py:49-97)."""

    ns: tuple
    samples: tuple
    nq: int
    p_vac: float
    delta: float

    def __post_init__(self):
        if not self.ns:
            raise ValueError("level plan needs at least one level")
        if len(self.ns) != len(self.samples):
            raise ValueError("ns and samples must have matching lengths")
        for n in self.ns:
            if n < 1:
                raise ValueError(f"supercell factor must be >= 1, got {n}")
        for a, b in zip(self.ns, self.ns[1:]):
            if b != 2 * a:
                raise ValueError(f"level sizes must double: {self.ns}")
        for m in self.samples:
            if m < 1:
                raise ValueError(f"sample counts must be >= 1, got {m}")
        if not 0.0 <= self.p_vac <= 1.0:
            raise ValueError(f"p_vac must be in [0, 1], got {self.p_vac}")
        if self.delta <= 0:
            raise ValueError("smoothing width must be positive")
        for n in self.ns:
            if self.q(n) < 1:
                raise ValueError(f"n*q = {self.nq} gives no k-points at n = {n}")

    @classmethod
    def geometric(cls, c: int, num_levels: int, **kw) -> "LevelPlan":
        return cls(ns=tuple(c * 2**lv for lv in range(1, num_levels + 1)), **kw)

    @property
    def num_levels(self) -> int:
        return len(self.ns)

    def q(self, n: int) -> int:
        if self.nq % n:
            raise ValueError(f"n*q constant {self.nq} not divisible by n = {n}")
        return self.nq // n


@dataclass(frozen=True, eq=False)
class LevelStats:
    level: int
    n: int
    q: int
    nsamples: int
    mean: np.ndarray = field(repr=False)
    sample_variance: np.ndarray | None = field(repr=False, default=None)
    work_per_sample: float = 0.0
    wall_seconds: float = 0.0
    cache_hits: int = 0


@dataclass(frozen=True, eq=False)
class MlmcEstimate:
    grid: object
    mean: np.ndarray = field(repr=False)
    estimator_variance: np.ndarray | None = field(repr=False)
    levels: tuple = ()
    total_wall_seconds: float = 0.0

    def level_window_variances(self, window=None):
        mask = window_mask(self.grid, window)
        return [float(np.mean(ls.sample_variance[mask])) if ls.sample_variance is not None else math.nan
                for ls in self.levels]


def window_mask(grid, window=None) -> np.ndarray:
    if window is None:
        return np.ones(grid.npoints, dtype=bool)
    lo, hi = window
    v = grid.values
    mask = (v >= lo) & (v <= hi)
    if not mask.any():
        raise ValueError(f"energy window {window} contains no grid points")
    return mask


def level_moments(full, quarters=None, device: int = 0, want_terms: bool = True):
    """(terms, mean, var) on the GPU; `full` [M, npts], `quarters` [M, 4, npts] or None.

    Accepts numpy arrays or CUDA torch tensors; returns torch tensors on the device (terms None when
    want_terms is False).  Host arrays go up through pinned staging (asynchronous DMA on the moments stream).
    """
    import torch

    dev = torch.device("cuda", device)
    # a high-priority stream: a level's moments are short and run while the later levels' solves still
    # occupy the SMs - the priority puts their blocks ahead of the queued solve blocks
    st = _moments_stream(device)
    st.wait_stream(torch.cuda.current_stream(dev))

    host = [a for a in (full, quarters) if a is not None and not isinstance(a, torch.Tensor)]
    stage = _pinned_staging(device, sum(int(np.asarray(a).size) for a in host)) if host else None
    off = [0]

    def up(a):
        if isinstance(a, torch.Tensor):
            return a.to(dev, dtype=torch.float64).contiguous()
        a = np.ascontiguousarray(a, dtype=np.float64)
        h = stage[0][off[0]: off[0] + a.size]
        off[0] += a.size
        h.numpy()[:] = a.reshape(-1)
        return h.to(dev, non_blocking=True).view(a.shape)

    with torch.cuda.stream(st):
        f = up(full)
        M, npts = f.shape
        q = None if quarters is None else up(quarters)
        if stage is not None:
            stage[1].record(st)  # the staging buffer is free again once these copies are done
        terms = torch.empty_like(f) if want_terms else None
        mean = torch.empty(npts, dtype=torch.float64, device=dev)
        var = torch.empty(npts, dtype=torch.float64, device=dev)
        _lib.Device.ctx(device)
        _lib.check(_lib.load().hx_level_moments_device(f.data_ptr(), 0 if q is None else q.data_ptr(), M, npts,
                                                       0 if terms is None else terms.data_ptr(), mean.data_ptr(),
                                                       var.data_ptr(), st.cuda_stream),
                   "hx_level_moments_device")
    torch.cuda.current_stream(dev).wait_stream(st)
    return terms, mean, var


_MOMENT_STREAMS: dict = {}
_PINNED: dict = {}


def _pinned_staging(device: int, count: int):
    """(pinned float64 host buffer of >= count elements, event of its last copy) for `device`, reused across
    calls (pin_memory() per call measured ~3 ms each in the Engine's level finish); waits for the previous
    copy out of it before handing it out again."""
    import torch

    buf, ev = _PINNED.get(device, (None, None))
    if buf is None or buf.numel() < count:
        if ev is not None:
            ev.synchronize()
        buf = torch.empty(max(count, 1 << 20), dtype=torch.float64).pin_memory()
        ev = torch.cuda.Event()
        _PINNED[device] = (buf, ev)
    else:
        ev.synchronize()
    return buf, ev


def _moments_stream(device: int):
    import torch

    st = _MOMENT_STREAMS.get(device)
    if st is None:
        st = _MOMENT_STREAMS[device] = torch.cuda.Stream(device=device, priority=-1)
    return st


def exact_level_moments(full, quarters, m_total: int, allreduce=None):
    """Level (mean, var) over samples spread across ranks or devices, bitwise independent of the split.

    `full` [M, npts] and `quarters` [M, 4, npts] (or None) are this rank's samples - CUDA tensors (device
    kernels) or numpy arrays (host twins); `m_total` is the level's sample count over all ranks;
    `allreduce(int64 limbs)` sums the fixed-point limbs over the ranks in place (e.g. torch.distributed
    all_reduce with NCCL / gloo; None = single rank).  Two passes as np.var (mlmc.py:143-154): the exact sum
    of the terms gives the mean, then the exact sum of squared deviations from that mean gives the unbiased
    variance (NaN for m_total < 2).  With one rank the result equals hx_level_moments_device's bit for bit."""
    import torch

    if isinstance(full, torch.Tensor) and full.is_cuda:
        dev = full.device
        st = torch.cuda.current_stream(dev).cuda_stream
        lib = _lib.load()
        M, npts = full.shape
        f = full.contiguous()
        q = None if quarters is None else quarters.contiguous()
        limbs = torch.empty((npts, _lib.HX_FX_LIMBS), dtype=torch.int64, device=dev)
        mean = torch.empty(npts, dtype=torch.float64, device=dev)
        var = torch.empty(npts, dtype=torch.float64, device=dev)

        def sums(center):
            _lib.check(lib.hx_level_sums_fixed_device(f.data_ptr(), 0 if q is None else q.data_ptr(), M, npts,
                                                      0 if center is None else center.data_ptr(),
                                                      limbs.data_ptr(), st), "hx_level_sums_fixed_device")
            if allreduce is not None:
                allreduce(limbs)

        sums(None)
        _lib.check(lib.hx_fixed_finalize_device(limbs.data_ptr(), npts, float(m_total), mean.data_ptr(), st),
                   "hx_fixed_finalize_device")
        sums(mean)
        _lib.check(lib.hx_fixed_finalize_device(limbs.data_ptr(), npts, float(m_total - 1), var.data_ptr(), st),
                   "hx_fixed_finalize_device")
        return mean, var

    def host_reduce(x):
        if allreduce is None:
            return x
        t = torch.from_numpy(x)
        allreduce(t)
        return t.numpy()

    s1 = host_reduce(_lib.fixed_sums(full, quarters))
    mean = _lib.fixed_finalize(s1, m_total)
    s2 = host_reduce(_lib.fixed_sums(full, quarters, mean))
    return mean, _lib.fixed_finalize(s2, m_total - 1)


def mean_and_variance(curves):
    """Pointwise mean and unbiased variance over axis 0; variance None for one sample (mlmc.py:143-154)."""
    curves = np.asarray(curves)
    if curves.ndim != 2 or curves.shape[0] < 1:
        raise ValueError("expected a (nsamples, npoints) array")
    _, mean, var = level_moments(curves)
    mean = mean.cpu().numpy()
    return (mean, None) if curves.shape[0] < 2 else (mean, var.cpu().numpy())


def control_variate_sample(config, partition, evaluate_full, evaluate_quarter):
    """Coupled (Q_l, Q_l^CV) for one outcome (mlmc.py:157-174)."""
    from .sampling import restrict

    q_full = np.asarray(evaluate_full(config))
    acc = None
    for r in range(1, partition.R + 1):
        part = np.asarray(evaluate_quarter(restrict(config, partition, r)))
        acc = part.copy() if acc is None else acc + part
    return q_full, acc / partition.R


def combine_levels(grid, levels, total_wall_seconds: float = 0.0) -> MlmcEstimate:
    """Sum of level means; estimator variance sum_l V_l / M_l (mlmc.py:177-196)."""
    if not levels:
        raise ValueError("no levels to combine")
    mean = np.zeros(grid.npoints)
    var = np.zeros(grid.npoints)
    ok = True
    for ls in levels:
        mean = mean + ls.mean
        if ls.sample_variance is None:
            ok = False
        else:
            var = var + ls.sample_variance / ls.nsamples
    return MlmcEstimate(grid=grid, mean=mean, estimator_variance=var if ok else None, levels=tuple(levels),
                        total_wall_seconds=total_wall_seconds)


# ---- rate fits of the "rates" mode (mlmc.py:260-338): host arithmetic on a handful of level statistics --------
@dataclass(frozen=True)
class RateFit:
    value: float
    stderr: float

    def __float__(self):
        return self.value


def fit_loglog_slope(sizes, observations) -> RateFit:
    """Least-squares slope of log(observation) on log(size) with its standard error (NaN for two points)
    (mlmc.py:268-285)."""
    x = np.log(np.asarray(sizes, dtype=float))
    y = np.asarray(observations, dtype=float)
    if np.any(y <= 0):
        raise ValueError("observations must be positive for a log-log fit")
    if len(x) != len(y) or len(x) < 2:
        raise ValueError("need at least two (size, observation) pairs")
    y = np.log(y)
    xc = x - x.mean()
    sxx = float(np.dot(xc, xc))
    slope = float(np.dot(xc, y) / sxx)
    se = math.nan
    if len(x) > 2:
        r = y - (y.mean() + slope * xc)
        se = math.sqrt(float(np.dot(r, r)) / (len(x) - 2) / sxx)
    return RateFit(slope, se)


@dataclass(frozen=True)
class RateEstimates:
    """Exponents: bias W, variance S, CV-difference variance D (decays, positive) and cost C (growth)
    (mlmc.py:288-303)."""

    w: RateFit | None = None
    s: RateFit | None = None
    d: RateFit | None = None
    c: RateFit | None = None

    @property
    def mlmc_benefit(self) -> bool:
        return self.d is not None and self.s is not None and self.d.value > self.s.value

    @property
    def mc_benefit(self) -> bool:
        return self.c is not None and self.s is not None and self.c.value > self.s.value


def fit_rates(sizes, bias_proxies=None, variances=None, cv_diff_variances=None, work=None) -> RateEstimates:
    """Model exponents from per-level observations; bias proxies |mean_l - mean_{l+1}| pair with sizes[:-1]
    (mlmc.py:306-338)."""
    sizes = tuple(int(n) for n in sizes)
    if len(sizes) < 2:
        raise ValueError("need at least two levels to fit rates")

    def decay(obs, xs):
        f = fit_loglog_slope(xs, obs)
        return RateFit(-f.value, f.stderr)

    w = None if bias_proxies is None else decay(tuple(bias_proxies), sizes[: len(tuple(bias_proxies))])
    s = None if variances is None else decay(variances, sizes)
    d = None if cv_diff_variances is None else decay(cv_diff_variances, sizes)
    c = None if work is None else fit_loglog_slope(sizes, work)
    return RateEstimates(w=w, s=s, d=d, c=c)
