"""Tight-binding models and their compiled supercell coupling tables (host side).

Mirrors tbmodel.py:40-146 (models), :162-221 (coupling expansion), :321-385 (table files).  The
dense Bloch assembly itself runs on the GPU (hx_assemble_device / the fused solve kernels); this
module only prepares the per-(model, n) instance tables in the reference's instance order, grouped
by source dof (CSR), and decides the pencil kind:
  * GrapheneNNModel -> commuting pencil: H = eps_2p I + t T, S = I + s T with one phase matrix T,
    so eps = (eps_2p + t*lam)/(1 + s*lam) for the eigenvalues lam of T (exact; SURVEY finding 2);
  * table without overlap couplings -> standard Hermitian problem (zheevd, spectrum.py:103);
  * table with overlap couplings -> general pencil via Cholesky (zhegv, spectrum.py:106-108).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .geometry import LatticeSpec, Supercell, honeycomb

__all__ = ["GrapheneNNModel", "MultiOrbitalModel", "BlochOperatorPair", "CompiledCell", "compile_cell",
           "assemble_bloch", "hermiticity_check", "load_coupling_table"]

GRAPHENE_EPS_2P = 0.0
GRAPHENE_T = -3.033
GRAPHENE_S = 0.129
MAX_COUPLING_RANGE = 3


@dataclass(frozen=True)
class GrapheneNNModel:
    """Nearest-neighbour pi-band model (tbmodel.py:40-79)."""

    eps_2p: float = GRAPHENE_EPS_2P
    t: float = GRAPHENE_T
    s: float = GRAPHENE_S

    def __post_init__(self):
        if abs(3.0 * self.s) >= 1.0:
            raise ValueError(f"overlap parameter s={self.s} makes S(k) singular")

    _NEIGHBOR_CELLS = ((0, 0), (-1, 0), (0, -1))

    def key(self):
        return ("graphene", self.eps_2p, self.t, self.s)

    def lattice_spec(self) -> LatticeSpec:
        return honeycomb()

    @property
    def overlap_is_identity(self) -> bool:
        return False

    def _entries(self, amp):
        fwd = [(di, dj, 0, 0, 1, 0, complex(amp)) for di, dj in self._NEIGHBOR_CELLS]
        return tuple(fwd + [(-di, -dj, 1, 0, 0, 0, complex(amp)) for di, dj in self._NEIGHBOR_CELLS])

    def hop_entries(self):
        return self._entries(self.t)

    def overlap_entries(self):
        return self._entries(self.s)

    def onsite_energies(self):
        return ((0, 0, self.eps_2p), (1, 0, self.eps_2p))


def _check_hermitian_closure(entries, what):
    sums = {}
    for di, dj, bs, os_, bd, od, amp in entries:
        k = (di, dj, bs, os_, bd, od)
        sums[k] = sums.get(k, 0.0) + complex(amp)
    for (di, dj, bs, os_, bd, od), amp in sums.items():
        mirror = sums.get((-di, -dj, bd, od, bs, os_))
        if mirror is None or abs(np.conj(mirror) - amp) > 1e-12 * max(1.0, abs(amp)):
            raise ValueError(f"{what} table not closed under Hermitian conjugation at "
                             f"displacement ({di},{dj}) basis {bs}/{os_} -> {bd}/{od}")


@dataclass(frozen=True)
class MultiOrbitalModel:
    """Table-driven honeycomb model (tbmodel.py:96-146)."""

    orbitals: tuple
    onsite: tuple
    hops: tuple
    overlap: tuple | None = None
    removable: tuple = ("B",)
    label: str = "table"

    def __post_init__(self):
        counts = dict(self.orbitals)
        for entries, what in ((self.hops, "hopping"), (self.overlap or (), "overlap")):
            for di, dj, bs, os_, bd, od, _ in entries:
                if max(abs(di), abs(dj)) > MAX_COUPLING_RANGE:
                    raise ValueError(f"{what} displacement ({di},{dj}) beyond third neighbors")
                if (di, dj) == (0, 0) and (bs, os_) == (bd, od):
                    raise ValueError(f"{what} entry duplicates an on-site term")
            _check_hermitian_closure(entries, what)
        roles = [r for r, _ in self.orbitals]
        for b, o, _ in self.onsite:
            if not 0 <= b < len(roles) or not 0 <= o < counts[roles[b]]:
                raise ValueError(f"on-site term for unknown orbital ({b},{o})")

    def key(self):
        return ("multiorbital", self.orbitals, self.onsite, self.hops, self.overlap, self.removable)

    def lattice_spec(self) -> LatticeSpec:
        return honeycomb(orbitals=self.orbitals, removable_roles=self.removable)

    @property
    def overlap_is_identity(self) -> bool:
        return self.overlap is None

    def hop_entries(self):
        return self.hops

    def overlap_entries(self):
        return self.overlap

    def onsite_energies(self):
        return self.onsite


@dataclass(frozen=True, eq=False)
class BlochOperatorPair:
    k: tuple
    H: np.ndarray = field(repr=False)
    S: np.ndarray = field(repr=False)
    dof_index: tuple = field(repr=False)


def _expand(sc: Supercell, site_offset: np.ndarray, entries):
    """Instances (src_dof, dst_dof, amp, disp) in reference order: sites, then table order (tbmodel.py:198-221)."""
    if not entries:
        z = np.zeros(0, dtype=np.int64)
        return z, z, np.zeros(0, dtype=np.complex128), np.zeros((0, 2))
    spec = sc.spec
    a = spec.vectors
    frac = spec.frac
    ent = np.array([(e[0], e[1], e[2], e[3], e[4], e[5]) for e in entries], dtype=np.int64)
    amp = np.array([complex(e[6]) for e in entries], dtype=np.complex128)
    # (site, entry) pairs where the entry's source basis matches the site's basis, site-major
    match = sc.basis_index[:, None] == ent[None, :, 2]
    s_idx, e_idx = np.nonzero(match)  # row-major: site-major then entry order
    i = sc.cells[s_idx, 0] + ent[e_idx, 0]
    j = sc.cells[s_idx, 1] + ent[e_idx, 1]
    sd = sc.site_index(i, j, ent[e_idx, 4])
    src = site_offset[s_idx] + ent[e_idx, 3]
    dst = site_offset[sd] + ent[e_idx, 5]
    v = (ent[e_idx, :2].astype(float) + frac[ent[e_idx, 4]]) - frac[ent[e_idx, 2]]
    disp = np.stack([v[:, 0] * a[0, 0] + v[:, 1] * a[1, 0], v[:, 0] * a[0, 1] + v[:, 1] * a[1, 1]], axis=1)
    return src.astype(np.int64), dst.astype(np.int64), amp[e_idx], disp


def _csr(n, src, dst, amp, disp):
    order = np.argsort(src, kind="stable")
    ptr = np.zeros(n + 1, dtype=np.int32)
    np.add.at(ptr, src + 1, 1)
    ptr = np.cumsum(ptr).astype(np.int32)
    a = np.ascontiguousarray(np.stack([amp.real, amp.imag], axis=1)[order].reshape(-1))
    dsp = np.ascontiguousarray(disp[order].reshape(-1))
    return ptr, np.ascontiguousarray(dst[order], dtype=np.int32), a, dsp


class CompiledCell:
    """Model couplings expanded on one supercell, uploaded once to the GPU (tbmodel.py:162-224)."""

    def __init__(self, model, supercell: Supercell, device: int = 0):
        self.model = model
        self.supercell = supercell
        counts = supercell.orbital_counts()
        self.site_offset = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
        self.dim = int(self.site_offset[-1])
        self.dof_site = np.repeat(np.arange(supercell.nsites), counts)
        self.dof_orb = np.concatenate([np.arange(c) for c in counts]) if self.dim else np.zeros(0, np.int64)
        self.onsite = np.zeros(self.dim)
        for b, o, e in model.onsite_energies():
            sites = np.flatnonzero(supercell.basis_index == b)
            self.onsite[self.site_offset[sites] + o] = e
        self.unit_of_dof = np.full(self.dim, -1, dtype=np.int32)
        self.unit_dofs = []
        for u, group in enumerate(supercell.removable_units):
            dofs = np.concatenate([np.arange(self.site_offset[s], self.site_offset[s + 1]) for s in group])
            self.unit_of_dof[dofs] = u
            self.unit_dofs.append(dofs)
        self.unit_dofs = tuple(self.unit_dofs)
        self.h = _expand(supercell, self.site_offset, model.hop_entries())
        ov = model.overlap_entries()
        self.s = None if ov is None else _expand(supercell, self.site_offset, ov)
        self.pencil, self.pencil_params = self._pencil_kind()
        self.device = device
        self._handle = None

    @property
    def time_reversal_symmetric(self) -> bool:
        """Real hopping / overlap amplitudes and on-site terms: H(-k) = conj(H(k)), S(-k) = conj(S(k)), so k
        and -k share a spectrum (the IDOS batches merge them, solver.time_reversal_reduce)."""
        amps = [np.asarray(self.h[2])] + ([] if self.s is None else [np.asarray(self.s[2])])
        return all(not np.any(np.imag(a)) for a in amps) and not np.any(np.imag(self.onsite))

    def _pencil_kind(self):
        m = self.model
        if isinstance(m, GrapheneNNModel) and m.t != 0.0:
            return _lib.HX_PENCIL_COMMUTING, (m.eps_2p, m.t, m.s)
        if self.s is None:
            return _lib.HX_PENCIL_STANDARD, (0.0, 1.0, 0.0)
        return _lib.HX_PENCIL_GENERAL, (0.0, 1.0, 0.0)

    @property
    def handle(self):
        """Device-resident copy (hx_cell*), created on first use."""
        if self._handle is None:
            lib = _lib.load()
            ctx = _lib.Device.ctx(self.device)
            src, dst, amp, disp = self.h
            if self.pencil == _lib.HX_PENCIL_COMMUTING:
                amp = amp / self.pencil_params[1]
            hp, hc, ha, hd = _csr(self.dim, src, dst, amp, disp)
            keep = [hp, hc, ha, hd]
            desc = _lib.CellDesc()
            desc.ndof = self.dim
            desc.nunits = self.supercell.nunits
            uod = np.ascontiguousarray(self.unit_of_dof, dtype=np.int32)
            ons = np.ascontiguousarray(self.onsite, dtype=np.float64)
            keep += [uod, ons]
            desc.unit_of_dof, desc.onsite = _lib.ptr(uod), _lib.ptr(ons)
            desc.h_row_ptr, desc.h_col, desc.h_amp, desc.h_disp = (_lib.ptr(x) for x in (hp, hc, ha, hd))
            if self.pencil == _lib.HX_PENCIL_GENERAL:
                sp, sc_, sa, sd = _csr(self.dim, *self.s)
                keep += [sp, sc_, sa, sd]
                desc.s_row_ptr, desc.s_col, desc.s_amp, desc.s_disp = (_lib.ptr(x) for x in (sp, sc_, sa, sd))
            desc.pencil = self.pencil
            desc.eps0, desc.t, desc.s = self.pencil_params
            desc.area = float(self.supercell.area)
            sub = np.ascontiguousarray(self.supercell.basis_index[self.dof_site], dtype=np.int32)
            keep.append(sub)
            desc.sublattice = _lib.ptr(sub)
            pos = np.ascontiguousarray(self.supercell.positions[self.dof_site], dtype=np.float64).reshape(-1)
            keep.append(pos)
            desc.dof_pos = _lib.ptr(pos)
            h = C.c_void_p()
            _lib.check(lib.hx_cell_create(ctx, C.byref(desc), C.byref(h)), "hx_cell_create")
            self._handle = h
            self._keep = keep
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _lib._lib is not None:
            try:
                _lib._lib.hx_cell_destroy(h)
            except Exception:  # noqa: BLE001 - interpreter teardown
                pass

    def configure(self, vacant_units=()):
        keep = np.ones(self.dim, dtype=bool)
        for u in vacant_units:
            keep[self.unit_dofs[u]] = False
        if not keep.any():
            raise ValueError("empty system: all orbitals removed by vacancies")
        return keep

    def kept_dims(self, words: np.ndarray) -> np.ndarray:
        """Kept dimension d of each uint64 mask row [R, w] (N minus the dofs of the vacant units)."""
        words = np.ascontiguousarray(words, dtype=np.uint64)
        bits = np.unpackbits(words.view(np.uint8), axis=1, bitorder="little")[:, : self.supercell.nunits]
        per_unit = np.array([len(d) for d in self.unit_dofs], dtype=np.int64)
        return self.dim - bits.astype(np.int64) @ per_unit

    def mask_words(self, vacant_units) -> np.ndarray:
        words = max(1, (self.supercell.nunits + 63) // 64)
        out = np.zeros(words, dtype=np.uint64)
        for u in vacant_units:
            out[u >> 6] |= np.uint64(1) << np.uint64(u & 63)
        return out


def compile_cell(model, supercell: Supercell, device: int = 0) -> CompiledCell:
    return CompiledCell(model, supercell, device)


def assemble_bloch(model, supercell: Supercell, defects, k) -> BlochOperatorPair:
    """H(k), S(k) with vacant rows/columns removed, assembled on the GPU (tbmodel.py:277-293)."""
    k = np.asarray(k, dtype=float)
    if k.shape != (2,) or not np.all(np.isfinite(k)):
        raise ValueError(f"k must be a finite 2-vector, got {k!r}")
    vacant = () if defects is None else defects.vacant
    cell = compile_cell(model, supercell)
    keep = cell.configure(vacant)
    import torch

    N = cell.dim
    dev = torch.device("cuda", cell.device)
    masks = torch.from_numpy(cell.mask_words(vacant).reshape(1, -1).view(np.int64)).to(dev)
    H = torch.zeros((N, N, 2), dtype=torch.float64, device=dev)
    S = torch.zeros((N, N, 2), dtype=torch.float64, device=dev)
    dims = torch.zeros(1, dtype=torch.int32, device=dev)
    kp = np.ascontiguousarray(k.reshape(1, 2))
    _lib.check(_lib.load().hx_assemble_device(_lib.Device.ctx(cell.device), cell.handle, _lib.ptr(kp), 1,
                                             masks.data_ptr(), 1, H.data_ptr(), S.data_ptr(), dims.data_ptr(),
                                             torch.cuda.current_stream(dev).cuda_stream), "hx_assemble_device")
    d = int(dims.item())
    # device layout is column-major N x N complex; take the leading d x d block
    Hc = torch.view_as_complex(H).cpu().numpy().T[:d, :d].copy()
    Sc = torch.view_as_complex(S).cpu().numpy().T[:d, :d].copy()
    dof_index = tuple((int(s), int(o)) for s, o in zip(cell.dof_site[keep], cell.dof_orb[keep]))
    return BlochOperatorPair(k=(float(k[0]), float(k[1])), H=Hc, S=Sc, dof_index=dof_index)


def hermiticity_check(pair: BlochOperatorPair) -> float:
    return float(np.max(np.abs(pair.H - pair.H.conj().T))) if pair.H.size else 0.0


_ROLE = {"A": 0, "B": 1}


def load_coupling_table(path) -> MultiOrbitalModel:
    """Parse a 'tbcoupling v1' file (format and errors as tbmodel.py:301-385)."""
    orbitals, onsite, hops, ovl = {}, [], [], []
    ident = False
    removable = None
    header = False

    def fail(lineno, msg):
        raise ValueError(f"{path}:{lineno}: {msg}")

    with open(path, encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            if not header:
                if line != "tbcoupling v1":
                    fail(lineno, f"expected header 'tbcoupling v1', got {line!r}")
                header = True
                continue
            tok = line.split()
            kind = tok[0]
            try:
                if kind == "orbitals":
                    orbitals[tok[1]] = int(tok[2])
                elif kind == "removable":
                    removable = tuple(tok[1:])
                elif kind == "onsite":
                    onsite.append((_ROLE[tok[1]], int(tok[2]), float(tok[3])))
                elif kind == "overlap":
                    if tok[1] != "identity":
                        fail(lineno, "only 'overlap identity' is supported here")
                    ident = True
                elif kind in ("coupling", "overlap_coupling"):
                    e = (int(tok[1]), int(tok[2]), _ROLE[tok[3]], int(tok[4]), _ROLE[tok[5]], int(tok[6]),
                         complex(float(tok[7]), float(tok[8])))
                    (hops if kind == "coupling" else ovl).append(e)
                else:
                    fail(lineno, f"unknown directive {kind!r}")
            except (IndexError, KeyError, ValueError) as exc:
                if isinstance(exc, ValueError) and str(exc).startswith(str(path)):
                    raise
                fail(lineno, f"malformed {kind!r} line: {exc}")
    if not header:
        raise ValueError(f"{path}: empty coupling table")
    if set(orbitals) != {"A", "B"}:
        raise ValueError(f"{path}: orbital counts must be given for roles A and B")
    if ovl and ident:
        raise ValueError(f"{path}: both 'overlap identity' and overlap couplings given")
    return MultiOrbitalModel(orbitals=(("A", orbitals["A"]), ("B", orbitals["B"])), onsite=tuple(onsite),
                             hops=tuple(hops), overlap=None if (ident or not ovl) else tuple(ovl),
                             removable=("B",) if removable is None else removable, label=str(path))
