"""CPU oracle for the hexmc hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain numpy/scipy restatement of the reference algorithm for the per-sample
supercell solve (geometry -> coupling expansion -> vacancy compaction -> Bloch H(k), S(k) ->
LAPACK eigenvalues -> smoothed/sharp IDOS -> level moments).  It exists so that `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / reference legs can CHECK the CUDA
product path.  The product package (`paper_1611_09784_b200`) never imports it.

Parity pin: every function here is checked against fixtures produced by running the reference
itself (`oracle/make_golden.py` -> `tests/golden/*.npz`) in `tests/test_oracle_golden.py`.

Reference citations are `path:line` into the reference package `pkg/src/hexmc/`.
Third-party arithmetic the reference calls (and therefore this oracle calls too):
  * LAPACK zhegv / zheevd through scipy 1.18 / numpy 2.3 (scipy-openblas 0.3.30)
    — reference call sites spectrum.py:103, spectrum.py:106-108.
  * numpy SeedSequence + PCG64 + Generator.random (numpy 2.3.5) — disorder.py:66-68, :79.
    `seedseq_pcg64_uniforms` below restates that published algorithm in pure Python so the
    product's C port can be pinned against it as well as against numpy.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg

# --- model constants (tbmodel.py:33-35) ---------------------------------------------------------
GRAPHENE_EPS_2P = 0.0
GRAPHENE_T = -3.033
GRAPHENE_S = 0.129
SLMC_STREAM_OFFSET = 10_000  # runner.py:53


# --- geometry (lattice.py:92-106, 160-195) ------------------------------------------------------
def honeycomb_vectors():
    """a1, a2 rows and basis fractional coordinates (lattice.py:97-106)."""
    r = 0.5 * np.sqrt(3.0)
    a = np.array([[r, 0.5], [r, -0.5]])
    frac = np.array([[0.0, 0.0], [1.0 / 3.0, 1.0 / 3.0]])
    return a, frac


def reciprocal(a):
    """b1, b2 with a_i.b_j = 2 pi delta_ij (lattice.py:81-86)."""
    det = a[0, 0] * a[1, 1] - a[0, 1] * a[1, 0]
    b1 = 2.0 * np.pi * np.array([a[1, 1], -a[1, 0]]) / det
    b2 = 2.0 * np.pi * np.array([-a[0, 1], a[0, 0]]) / det
    return b1, b2


class Cell:
    """n x n supercell; site s = (i*n + j)*2 + b (lattice.py:139-141, 173-177)."""

    def __init__(self, n, orbitals=(1, 1), removable=(0, 1), n2=None):
        # n2: cells along a2 of a rectangular n x n2 supercell (the package's config-5 extension; the reference
        # builds square cells only, lattice.py:160-195, so rectangular parity rests on this same restatement)
        self.n = n
        self.m = n if n2 is None else n2
        self.orbitals = tuple(orbitals)
        ii, jj, bb = np.meshgrid(np.arange(n), np.arange(self.m), np.arange(2), indexing="ij")
        self.ci = ii.reshape(-1)
        self.cj = jj.reshape(-1)
        self.basis = bb.reshape(-1)
        self.nsites = 2 * n * self.m
        counts = np.array([orbitals[b] for b in self.basis])
        self.site_offset = np.concatenate(([0], np.cumsum(counts)))
        self.dim = int(self.site_offset[-1])
        self.unit_sites = np.array([s for s in range(self.nsites) if self.basis[s] in removable], dtype=np.int64)
        self.nunits = len(self.unit_sites)
        # unit_dofs, tbmodel.py:191-196
        self.unit_dofs = [np.arange(self.site_offset[s], self.site_offset[s + 1]) for s in self.unit_sites]
        self.area = float(n * self.m)  # normalized area (lattice.py:131-133, area_unit = cell area)

    def site_index(self, i, j, b):
        return ((i % self.n) * self.m + (j % self.m)) * 2 + b


# --- models (tbmodel.py:40-79, 321-385) ---------------------------------------------------------
def graphene_model(eps=GRAPHENE_EPS_2P, t=GRAPHENE_T, s=GRAPHENE_S):
    nbr = ((0, 0), (-1, 0), (0, -1))
    hops = [(di, dj, 0, 0, 1, 0, complex(t)) for di, dj in nbr] + [(-di, -dj, 1, 0, 0, 0, complex(t)) for di, dj in nbr]
    ovl = [(di, dj, 0, 0, 1, 0, complex(s)) for di, dj in nbr] + [(-di, -dj, 1, 0, 0, 0, complex(s)) for di, dj in nbr]
    return {
        "orbitals": (1, 1),
        "removable": (0, 1),
        "onsite": [(0, 0, eps), (1, 0, eps)],
        "hops": hops,
        "overlap": ovl,
    }


def parse_table(path):
    """Restatement of load_coupling_table (tbmodel.py:321-385) for the happy path."""
    roles = {"A": 0, "B": 1}
    orb = {}
    onsite, hops, ovl = [], [], []
    removable = None
    ident = False
    header = False
    for raw in open(path, encoding="utf-8"):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if not header:
            assert line == "tbcoupling v1"
            header = True
            continue
        tok = line.split()
        if tok[0] == "orbitals":
            orb[tok[1]] = int(tok[2])
        elif tok[0] == "removable":
            removable = tuple(tok[1:])
        elif tok[0] == "onsite":
            onsite.append((roles[tok[1]], int(tok[2]), float(tok[3])))
        elif tok[0] == "overlap":
            ident = True
        elif tok[0] in ("coupling", "overlap_coupling"):
            e = (int(tok[1]), int(tok[2]), roles[tok[3]], int(tok[4]), roles[tok[5]], int(tok[6]),
                 complex(float(tok[7]), float(tok[8])))
            (hops if tok[0] == "coupling" else ovl).append(e)
    return {
        "orbitals": (orb["A"], orb["B"]),
        "removable": tuple(roles[r] for r in (removable or ("B",))),
        "onsite": onsite,
        "hops": hops,
        "overlap": None if (ident or not ovl) else ovl,
    }


def make_cell(model, n, n2=None):
    return Cell(n, model["orbitals"], model["removable"], n2)


def expand(cell, entries):
    """Coupling instances per source site in site order (tbmodel.py:198-221)."""
    a, frac = honeycomb_vectors()
    src, dst, amp, disp = [], [], [], []
    for s in range(cell.nsites):
        b = cell.basis[s]
        for di, dj, bs, os_, bd, od, am in entries:
            if bs != b:
                continue
            sd = cell.site_index(cell.ci[s] + di, cell.cj[s] + dj, bd)
            src.append(cell.site_offset[s] + os_)
            dst.append(cell.site_offset[sd] + od)
            amp.append(am)
            disp.append((np.array([di, dj], dtype=float) + frac[bd] - frac[b]) @ a)
    return (np.array(src, dtype=np.int64), np.array(dst, dtype=np.int64),
            np.array(amp, dtype=np.complex128), np.array(disp, dtype=np.float64).reshape(-1, 2))


def onsite_vector(cell, model):
    v = np.zeros(cell.dim)
    for b, o, e in model["onsite"]:
        for s in np.flatnonzero(cell.basis == b):
            v[cell.site_offset[s] + o] = e
    return v


def keep_of_mask(cell, mask):
    """keep[] and compaction map (tbmodel.py:233-239)."""
    keep = np.ones(cell.dim, dtype=bool)
    for u in range(cell.nunits):
        if (mask >> u) & 1:
            keep[cell.unit_dofs[u]] = False
    return keep


def assemble(cell, model, mask, k):
    """Dense H(k), S(k) with vacant rows/cols removed (tbmodel.py:246-270, _kernels.py:62-65)."""
    keep = keep_of_mask(cell, mask)
    d = int(keep.sum())
    if d == 0:
        raise ValueError("empty system: all orbitals removed by vacancies")
    new = np.cumsum(keep) - 1
    k = np.asarray(k, dtype=float)

    def build(entries, diag):
        M = np.zeros((d, d), dtype=np.complex128)
        if entries is not None:
            src, dst, amp, disp = expand(cell, entries)
            for i in range(len(src)):
                if keep[src[i]] and keep[dst[i]]:
                    ph = disp[i, 0] * k[0] + disp[i, 1] * k[1]
                    M[new[src[i]], new[dst[i]]] += amp[i] * complex(math.cos(ph), math.sin(ph))
            M = 0.5 * (M + M.conj().T)
        M[np.diag_indices(d)] = diag
        return M

    H = build(model["hops"], onsite_vector(cell, model)[keep])
    S = build(model["overlap"], 1.0)
    return H, S


def eigvals(H, S, identity_overlap):
    """spectrum.py:100-117: zheevd for identity overlap, zhegv otherwise."""
    if identity_overlap:
        return np.linalg.eigvalsh(H)
    return scipy.linalg.eigh(H, S, eigvals_only=True, driver="gv", check_finite=False)


def bz_grid(n, q, mode="reduced"):
    """spectrum.py:59-84."""
    a, _ = honeycomb_vectors()
    b1, b2 = reciprocal(a)
    ii, jj = np.meshgrid(np.arange(q), np.arange(q), indexing="ij")
    base = ii.reshape(-1, 1) * (b1 / (n * q))[None, :] + jj.reshape(-1, 1) * (b2 / (n * q))[None, :]
    if mode == "reduced":
        kp = base
    else:
        def rot(t):
            return np.array([[np.cos(t), -np.sin(t)], [np.sin(t), np.cos(t)]])
        kp = np.concatenate([base, base @ rot(2.0 * np.pi / 3.0).T, base @ rot(4.0 * np.pi / 3.0).T])
    return kp, np.full(len(kp), 1.0 / len(kp))


def solve_bands(cell, model, mask, kpoints):
    """Per-k eigenvalues (spectrum.py:120-134)."""
    ident = model["overlap"] is None
    out = []
    for k in kpoints:
        H, S = assemble(cell, model, mask, k)
        out.append(eigvals(H, S, ident))
    return np.array(out)


# --- QoI (qoi.py:42-108, _kernels.py:68-101) ----------------------------------------------------
def grid_step(lo, hi, npts):
    return (hi - lo) / (npts - 1)


def smoothed_counts(E, w, e0, step, npts, delta):
    """Restates _kernels.py:68-88 (numba loop order)."""
    out = np.zeros(npts)
    suffix = np.zeros(npts + 1)
    for e, wt in zip(E, w):
        lo = int(math.ceil((e + delta - e0) / step))
        lo = max(lo, 0)
        if lo <= npts:
            suffix[lo] += wt
        m0 = max(int(math.floor((e - delta - e0) / step)) + 1, 0)
        m1 = min(lo, npts)
        for m in range(m0, m1):
            x = (e - (e0 + step * m)) / delta
            out[m] += wt * (0.5 + x * (-1.125 + 0.625 * x * x))
    out += np.cumsum(suffix[:npts])
    return out


def sharp_counts(E, w, e0, step, npts):
    """Restates _kernels.py:91-101."""
    suffix = np.zeros(npts + 1)
    for e, wt in zip(E, w):
        idx = max(int(math.floor((e - e0) / step)) + 1, 0)
        if idx <= npts:
            suffix[idx] += wt
    return np.cumsum(suffix[:npts])


def idos_from_bands(energies, kweights, lo, hi, npts, delta, area):
    """qoi.py:85-102."""
    nb = energies.shape[1]
    E = energies.reshape(-1)
    w = np.repeat(kweights, nb)
    return smoothed_counts(E, w, lo, grid_step(lo, hi, npts), npts, delta) / area


def idos_sharp_from_bands(energies, kweights, lo, hi, npts, area):
    nb = energies.shape[1]
    return sharp_counts(energies.reshape(-1), np.repeat(kweights, nb), lo, grid_step(lo, hi, npts), npts) / area


def sample_curve(model, n, q, mask, lo, hi, npts, delta, mode="reduced"):
    """One job of _eval_job (runner.py:114-129), including the all-vacant shortcut."""
    cell = make_cell(model, n)
    removed = sum(len(cell.unit_dofs[u]) for u in range(cell.nunits) if (mask >> u) & 1)
    if removed >= cell.dim:
        return np.zeros(npts)
    kp, kw = bz_grid(n, q, mode)
    bands = solve_bands(cell, model, mask, kp)
    return idos_from_bands(bands, kw, lo, hi, npts, delta, cell.area)


# --- disorder (disorder.py:40-94, lattice.py:222-259) -------------------------------------------
def numpy_uniforms(seed, level, rep, count):
    """The reference's draw (disorder.py:66-68, :79) via numpy itself."""
    g = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(level, rep)))
    return g.random(count)


_M32 = 0xFFFFFFFF
_M64 = (1 << 64) - 1
_M128 = (1 << 128) - 1
_PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def _words32(x):
    if x == 0:
        return [0]
    out = []
    while x > 0:
        out.append(x & _M32)
        x >>= 32
    return out


def seedseq_state(seed, spawn_key, nwords64=4):
    """Published numpy SeedSequence algorithm (pool of 4 uint32, hashmix/mix), restated."""
    ent = _words32(seed)
    spawn = [w for v in spawn_key for w in _words32(v)]
    if spawn and len(ent) < 4:
        ent = ent + [0] * (4 - len(ent))
    ent = ent + spawn
    hc = [0x43B0D7E5]

    def hashmix(v):
        v = (v ^ hc[0]) & _M32
        hc[0] = (hc[0] * 0x931E8875) & _M32
        v = (v * hc[0]) & _M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (0xCA01F9DD * x - 0x4973F715 * y) & _M32
        return r ^ (r >> 16)

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(4)]
    for i_src in range(4):
        for i_dst in range(4):
            if i_src != i_dst:
                pool[i_dst] = mix(pool[i_dst], hashmix(pool[i_src]))
    for i_src in range(4, len(ent)):
        for i_dst in range(4):
            pool[i_dst] = mix(pool[i_dst], hashmix(ent[i_src]))
    hb = 0x8B51F9DD
    st32 = []
    for i in range(2 * nwords64):
        v = pool[i % 4]
        v = (v ^ hb) & _M32
        hb = (hb * 0x58F38DED) & _M32
        v = (v * hb) & _M32
        v ^= v >> 16
        st32.append(v)
    return [st32[2 * i] | (st32[2 * i + 1] << 32) for i in range(nwords64)]


def seedseq_pcg64_uniforms(seed, level, rep, count):
    """Pure-Python PCG64 (XSL-RR 128/64) seeded like numpy's PCG64(SeedSequence); random()."""
    s = seedseq_state(seed, (level, rep), 4)
    initstate = (s[0] << 64) | s[1]
    inc = ((((s[2] << 64) | s[3]) << 1) | 1) & _M128
    state = 0
    state = (state * _PCG_MULT + inc) & _M128
    state = (state + initstate) & _M128
    state = (state * _PCG_MULT + inc) & _M128
    out = np.empty(count)
    for i in range(count):
        state = (state * _PCG_MULT + inc) & _M128
        hi, lo = state >> 64, state & _M64
        x = hi ^ lo
        r = state >> 122
        v = ((x >> r) | (x << ((64 - r) & 63))) & _M64
        out[i] = (v >> 11) * (1.0 / 9007199254740992.0)
    return out


def sample_mask(nunits, p, seed, level, rep):
    """disorder.py:71-81 -> canonical bitmask key (disorder.py:40-46)."""
    draws = numpy_uniforms(seed, level, rep, nunits)
    mask = 0
    for u in np.flatnonzero(draws < p):
        mask |= 1 << int(u)
    return mask


def quarter_maps(cell):
    """(unit_assignment, unit_map) of partition_quarters (lattice.py:222-259)."""
    n = cell.n
    h = n // 2
    sub = Cell(h, cell.orbitals, tuple(sorted(set(cell.basis[cell.unit_sites].tolist()))))
    sub_unit_of_site = -np.ones(sub.nsites, dtype=np.int64)
    sub_unit_of_site[sub.unit_sites] = np.arange(sub.nunits)
    assign = np.empty(cell.nunits, dtype=np.int64)
    umap = np.empty(cell.nunits, dtype=np.int64)
    for u, s in enumerate(cell.unit_sites):
        i, j, b = cell.ci[s], cell.cj[s], cell.basis[s]
        bi, bj = i // h, j // h
        assign[u] = 1 + 2 * bi + bj
        umap[u] = sub_unit_of_site[((i - bi * h) * h + (j - bj * h)) * 2 + b]
    return assign, umap


def restrict_mask(mask, assign, umap, r):
    """disorder.py:84-94 on bitmask keys."""
    out = 0
    for u in range(len(assign)):
        if (mask >> u) & 1 and assign[u] == r:
            out |= 1 << int(umap[u])
    return out


# --- estimator (mlmc.py:143-196, runner.py:254-311) ---------------------------------------------
def mean_and_variance(curves):
    curves = np.asarray(curves)
    mean = np.mean(curves, axis=0)
    if curves.shape[0] < 2:
        return mean, None
    return mean, np.var(curves, axis=0, ddof=1)


def sample_level(model, nq, level, n, nsamples, p, with_cv, seed, lo, hi, npts, delta, mode="reduced",
                 stream=None, cache=None):
    """Level terms with the quarter control variate (runner.py:254-311), dedup on (n, q, mask)."""
    cache = {} if cache is None else cache
    q = nq // n
    cell = make_cell(model, n)
    stream = level if stream is None else stream
    masks = [sample_mask(cell.nunits, p, seed, stream, m) for m in range(nsamples)]

    def curve(nn, qq, mk):
        key = (nn, qq, mk)
        if key not in cache:
            cache[key] = sample_curve(model, nn, qq, mk, lo, hi, npts, delta, mode)
        return cache[key]

    full = np.array([curve(n, q, mk) for mk in masks])
    cv = None
    if with_cv:
        assign, umap = quarter_maps(cell)
        cv = np.zeros_like(full)
        for m, mk in enumerate(masks):
            for r in range(1, 5):
                cv[m] += curve(n // 2, nq // (n // 2), restrict_mask(mk, assign, umap, r))
            cv[m] *= 0.25
    terms = full - cv if cv is not None else full
    mean, var = mean_and_variance(terms)
    return {"masks": masks, "full": full, "cv": cv, "terms": terms, "mean": mean, "variance": var}


def detect_energy_range(model, nq, mode="reduced"):
    """runner.py:189-202: unperturbed nu=1 band extrema on the q=nq grid."""
    cell = make_cell(model, 1)
    kp, _ = bz_grid(1, nq, mode)
    b = solve_bands(cell, model, 0, kp)
    return float(b.min()), float(b.max())
