"""GPU parity of every kernel variant the benchmark shapes select, against the oracle (LAPACK restatement).

The banded tiers pick their kernels from the batch size and the matrix size (hx_bdband.cu: real bulge chase
with 16 / 4 / 1 warps per matrix from ceil(1628 / matrices), padded shared memory for 2 <= want < 6,
clusters of 2-8 SMs per matrix for S >= 1024 ... 4096; real or complex storage; real Golub-Kahan at the
time-reversal-invariant k-points of the shared-memory tier).  Each test below either builds a batch of the
size the bench uses for that tier, or forces the variant through the option registry (hx_set_option, the
`_lib.options` context manager), and compares a subset of the batch with the oracle:
eigenvalues <= 1e-10 x spectral width, IDOS <= 1e-9 (BASELINE.json north_star).  Reference:
spectrum.py:100-134 (zhegv / zheevd per k), qoi.py:96-102 (IDOS).
"""

import numpy as np
import pytest

import hexmc_oracle as O
from conftest import TABLE, words_to_int

import paper_1611_09784_b200 as hx
from paper_1611_09784_b200 import _lib
from paper_1611_09784_b200.sampling import sample_masks
from paper_1611_09784_b200.solver import eval_batch

pytestmark = pytest.mark.gpu

EIG_TOL = 1e-10
IDOS_TOL = 1e-9
LO_G, HI_G = -6.580201874549387, 14.863393148450246
LO_T, HI_T = -2.952, 4.760
NPTS = 201


def _setup(kind, nu, q, kp=None):
    model = hx.load_coupling_table(TABLE) if kind == "table" else hx.GrapheneNNModel()
    om = O.parse_table(str(TABLE)) if kind == "table" else O.graphene_model()
    spec = model.lattice_spec()
    sc = hx.build_supercell(spec, nu)
    cell = hx.compile_cell(model, sc)
    if kp is None:
        kp = hx.make_bz_grid(spec, nu, q, "reduced").kpoints
    return model, om, sc, cell, np.ascontiguousarray(kp)


def check_batch(kind, nu, q, p, nmasks, seed, check, kp=None, opts=None, eigs_too=True):
    """Solve `nmasks` seeded masks in ONE batch (so the batch-size-dependent variant runs), compare the
    masks `check` with the oracle.  Both the eigenvalue path and the IDOS-only fast path are checked."""
    _, om, sc, cell, kp = _setup(kind, nu, q, kp)
    lo, hi = (LO_T, HI_T) if kind == "table" else (LO_G, HI_G)
    step = (hi - lo) / (NPTS - 1)
    words = sample_masks(sc.nunits, p, seed, 3, 0, nmasks)
    with _lib.options(**(opts or {})):
        fast, _, st_fast = eval_batch(cell, kp, words, lo, step, NPTS, 0.01)
        if eigs_too:
            curves, eigs, status = eval_batch(cell, kp, words, lo, step, NPTS, 0.01, want_eigs=True)
    assert (st_fast == 0).all()
    if eigs_too:
        assert (status == 0).all()
        np.testing.assert_allclose(fast, curves, rtol=0, atol=1e-11)
    ocell = O.make_cell(om, nu)
    for m in check:
        ref = O.solve_bands(ocell, om, words_to_int(words[m]), kp)
        d = ref.shape[1]
        if eigs_too:
            assert np.all(np.isnan(eigs[m, :, d:]))
            err = np.max(np.abs(eigs[m, :, :d] - ref))
            assert err <= EIG_TOL * (ref.max() - ref.min()), (m, err)
        rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), lo, hi, NPTS, 0.01, ocell.area)
        np.testing.assert_allclose(fast[m], rc, rtol=0, atol=IDOS_TOL)
    return fast


# ---- real bulge chase: every warps-per-matrix variant, forced (nu = 16, q = 2: S = 256, real batch) ----------
@pytest.mark.parametrize("reg", [1, 0])
@pytest.mark.parametrize("rnw", [1, 2, 4, 8, 16])
def test_real_chase_warp_variants_forced(rnw, reg):
    """Register-row chase (HX_CHASE_REG=1, default) and shared-memory-tile chase, every warps-per-matrix count."""
    check_batch("graphene", 16, 2, 0.05, 6, 31, (0, 5), opts={"HX_CHASE_RNW": rnw, "HX_CHASE_REG": reg})


# ---- the variants the c2 batch sizes select by themselves ----------------------------------------------------
@pytest.mark.parametrize("gram", [1, 0])
def test_real_chase_padded_nw4_at_bench_batch(gram):
    """c2 level 3 / level-4 quarters: 256 masks x 4 k = 1024 N = 512 matrices -> want = 2: the 4-warp chase at
    4-5 CTAs / SM - the symmetric chase of the Gram path (default for IDOS-only batches) and the bidiagonal chase of
    the SVD path (HX_GRAM=0).  8 masks spread over the batch are checked against the oracle."""
    check_batch("graphene", 16, 2, 0.05, 256, 2026, (0, 37, 101, 128, 170, 201, 240, 255), eigs_too=False,
                opts={"HX_GRAM": gram})


@pytest.mark.parametrize("gram", [1, 0])
def test_real_chase_nw1_at_large_batch(gram):
    """>= 1628 matrices -> want = 1: one warp per matrix (c5 n = 512 batches)."""
    check_batch("graphene", 16, 2, 0.05, 420, 7, (0, 211, 419), eigs_too=False, opts={"HX_GRAM": gram})


@pytest.mark.parametrize("gram", [1, 0])
def test_c2_level4_parent_batch(gram):
    """c2 level 4: 64 nu = 32 masks at Gamma (N = 2048, S = 1024) in one batch - the 8-warp chase (Gram path:
    half-task progress counters; SVD path: register-row bidiagonal chase)."""
    check_batch("graphene", 32, 1, 0.05, 64, 2026, (0, 33, 63), eigs_too=False, opts={"HX_GRAM": gram})


def test_clustered_real_chase_two_sms():
    """HX_CHASE_RCL = 2 (2 SMs per matrix) on S = 1024 (the default picks it from S >= 2048)."""
    check_batch("graphene", 32, 1, 0.05, 2, 5, (0, 1), opts={"HX_CHASE_RCL": 2})


@pytest.mark.parametrize("reg", [1, 0])
@pytest.mark.parametrize("rcl", [2, 4])
def test_clustered_real_chase_nu46(rcl, reg):
    check_batch("graphene", 46, 1, 0.02, 1, 9, (0,), opts={"HX_CHASE_RCL": rcl, "HX_CHASE_REG": reg})


# ---- real / complex storage and arithmetic switches -----------------------------------------------------------
@pytest.mark.parametrize("opts", [{"HX_NO_REAL": 1}, {"HX_REAL_STAGE1": 0}, {"HX_CHASE_REAL": 0}, {"HX_CHASE_REG": 0},
                                  {"HX_CHASE_PAIR": 0}, {"HX_REAL_FUSED": 1}, {"HX_FUSED_UPDATE": 1}])
@pytest.mark.parametrize("nu,q", [(16, 2), (12, 1), (11, 1)])
def test_real_path_switches(nu, q, opts):
    check_batch("graphene", nu, q, 0.1, 4, 13, (0, 3), opts=opts)


@pytest.mark.parametrize("opts", [{}, {"HX_BIDIAG_REAL": 0}, {"HX_NO_REAL": 1}, {"HX_NO_BIPARTITE": 1},
                                  {"HX_BIDIAG_REG": 0}])
@pytest.mark.parametrize("nu,q", [(4, 8), (8, 4), (8, 2)])
def test_shared_memory_tiers_switches(nu, q, opts):
    """The shared-memory tiers of c1/c2 (N = 32, 128): complex warp / CTA Golub-Kahan, real Golub-Kahan at the
    TRIM k-points, and the Hermitian (non-bipartite) tier with HX_NO_BIPARTITE."""
    check_batch("graphene", nu, q, 0.05, 40, 17, (0, 19, 39), opts=opts)


@pytest.mark.parametrize("reg", [1, 0])
@pytest.mark.parametrize("nu,q,conc", [(5, 3, 0.05), (6, 3, 0.2), (7, 5, 0.1), (8, 3, 0.3), (6, 4, 0.2), (7, 2, 0.1),
                                       (8, 2, 0.3)])
def test_register_golub_kahan(nu, q, conc, reg):
    """k-points with 32 < S <= 64 (N = 50..128): the register-resident 256-thread Golub-Kahan, complex and
    real (TRIM k, q = 2 / 4) (HX_BIDIAG_REG=1, default), and the shared-memory CTA / warp kernels, padded /
    rectangular blocks at high vacancy counts."""
    check_batch("graphene", nu, q, conc, 24, 23, (0, 11, 23), opts={"HX_BIDIAG_REG": reg})


# ---- complex bipartite banded tier (non-TRIM k, N > 160) ------------------------------------------------------
@pytest.mark.parametrize("opts", [{}, {"HX_RU_3M": 1}])
@pytest.mark.parametrize("nu,q", [(10, 3), (11, 4), (12, 3)])
def test_complex_bipartite_banded_tier(nu, q, opts):
    check_batch("graphene", nu, q, 0.05, 3, 21, (0, 2), opts=opts)


@pytest.mark.parametrize("nu", [16, 32])
def test_c5_generic_k_point(nu):
    """c5 sweep: one generic k (reduced q = 3 grid, point 4) per matrix at n = 512 and 2048."""
    kp = hx.make_bz_grid(hx.GrapheneNNModel().lattice_spec(), nu, 3, "reduced").kpoints[4:5]
    check_batch("graphene", nu, 1, 0.05, 4 if nu == 32 else 16, 2026, (0, 3), kp=kp)


# ---- c3 (11-band table, Hermitian banded tier) at the bench sizes ----------------------------------------------
def test_c3_table_nu8():
    check_batch("table", 8, 2, 0.05, 6, 2026, (0, 5))


def test_c3_table_nu16():
    check_batch("table", 16, 1, 0.05, 2, 2026, (0,))


# ---- c4 scale: a defected nu = 64 sample at Gamma against zhegv on the N = 8192 pencil -------------------------
def test_c4_defected_nu64_gamma():
    check_batch("graphene", 64, 1, 0.02, 1, 2026, (0,))


# ---- c5 sweep sizes on rectangular n x n2 supercells (n = 64, 256, 1024) --------------------------------------
@pytest.mark.parametrize("nu,nu2,count", [(4, 8, 64), (8, 16, 24), (16, 32, 4)])
def test_c5_rectangular_sizes(nu, nu2, count):
    model = hx.GrapheneNNModel()
    spec = model.lattice_spec()
    sc = hx.build_supercell(spec, nu, nu2)
    cell = hx.compile_cell(model, sc)
    b1, b2 = spec.reciprocal_vectors()
    kp = np.ascontiguousarray((b1 / (3 * nu) + b2 / (3 * nu2)).reshape(1, 2))
    step = (HI_G - LO_G) / (NPTS - 1)
    words = sample_masks(sc.nunits, 0.05, 2026, 5, 0, count)
    curves, eigs, status = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01, want_eigs=True)
    assert (status == 0).all()
    om = O.graphene_model()
    ocell = O.make_cell(om, nu, nu2)
    for m in (0, count - 1):
        ref = O.solve_bands(ocell, om, words_to_int(words[m]), kp)
        d = ref.shape[1]
        assert np.max(np.abs(eigs[m, :, :d] - ref)) <= EIG_TOL * (ref.max() - ref.min())
        rc = O.idos_from_bands(ref, np.ones(1), LO_G, HI_G, NPTS, 0.01, ocell.area)
        np.testing.assert_allclose(curves[m], rc, rtol=0, atol=IDOS_TOL)


# ---- general pencils above the shared-memory tier (overlap tables: Cholesky + banded two-stage) ---------------
def _general_models(kind):
    """(native model, oracle dict) of a pencil with overlap couplings (zhegv in the reference)."""
    if kind == "graphene":
        hops, ovl = [], []
        for di, dj in ((0, 0), (-1, 0), (0, -1)):
            ovl += [(di, dj, 0, 0, 1, 0, 0.129 + 0j), (-di, -dj, 1, 0, 0, 0, 0.129 + 0j)]
            hops += [(di, dj, 0, 0, 1, 0, -3.033 + 0j), (-di, -dj, 1, 0, 0, 0, -3.033 + 0j)]
        onsite = [(0, 0, 0.0), (1, 0, 0.0)]
        orbs, removable = (1, 1), ("A", "B")
    else:  # two orbitals per site, complex hops and overlaps, B removable
        rng = np.random.default_rng(12)
        hops, ovl = [], []
        for di, dj in ((0, 0), (-1, 0), (0, -1)):
            for oa in range(2):
                for ob in range(2):
                    h = complex(rng.normal(-1.0, 0.3), rng.normal(0, 0.2))
                    s = complex(rng.uniform(0.02, 0.06), rng.normal(0, 0.01))
                    hops += [(di, dj, 0, oa, 1, ob, h), (-di, -dj, 1, ob, 0, oa, h.conjugate())]
                    ovl += [(di, dj, 0, oa, 1, ob, s), (-di, -dj, 1, ob, 0, oa, s.conjugate())]
        onsite = [(0, 0, 0.3), (0, 1, 0.7), (1, 0, -0.2), (1, 1, 0.1)]
        orbs, removable = (2, 2), ("B",)
    model = hx.MultiOrbitalModel(orbitals=(("A", orbs[0]), ("B", orbs[1])), onsite=tuple(onsite), hops=tuple(hops),
                                 overlap=tuple(ovl), removable=removable)
    om = {"orbitals": orbs, "removable": tuple({"A": 0, "B": 1}[r] for r in removable), "onsite": onsite,
          "hops": hops, "overlap": ovl}
    return model, om


@pytest.mark.parametrize("kind,nu,q", [("graphene", 10, 1), ("graphene", 12, 2), ("twoorb", 7, 2), ("twoorb", 9, 1)])
def test_general_pencil_banded_tier(kind, nu, q):
    model, om = _general_models(kind)
    spec = model.lattice_spec()
    sc = hx.build_supercell(spec, nu)
    cell = hx.compile_cell(model, sc)
    assert cell.pencil == _lib.HX_PENCIL_GENERAL and cell.dim > 160
    kp = np.ascontiguousarray(hx.make_bz_grid(spec, nu, q, "reduced").kpoints)
    words = sample_masks(sc.nunits, 0.05, 2026, 3, 0, 3)
    lo, hi = -12.0, 14.0
    step = (hi - lo) / (NPTS - 1)
    curves, eigs, status = eval_batch(cell, kp, words, lo, step, NPTS, 0.01, want_eigs=True)
    assert (status == 0).all()
    ocell = O.make_cell(om, nu)
    for m in (0, 2):
        ref = O.solve_bands(ocell, om, words_to_int(words[m]), kp)
        d = ref.shape[1]
        assert np.max(np.abs(eigs[m, :, :d] - ref)) <= EIG_TOL * (ref.max() - ref.min())
        rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), lo, hi, NPTS, 0.01, ocell.area)
        np.testing.assert_allclose(curves[m], rc, rtol=0, atol=IDOS_TOL)
    with _lib.options(HX_GENERAL_BAND=0):  # the single-CTA global kernel agrees
        c2, _, _ = eval_batch(cell, kp, words, lo, step, NPTS, 0.01)
    np.testing.assert_allclose(c2, curves, rtol=0, atol=1e-10)


def test_general_pencil_banded_tier_non_pd_raises():
    hops, ovl = [], []
    for di, dj in ((0, 0), (-1, 0), (0, -1)):
        ovl += [(di, dj, 0, 0, 1, 0, 0.5 + 0j), (-di, -dj, 1, 0, 0, 0, 0.5 + 0j)]
        hops += [(di, dj, 0, 0, 1, 0, -1.0 + 0j), (-di, -dj, 1, 0, 0, 0, -1.0 + 0j)]
    model = hx.MultiOrbitalModel(orbitals=(("A", 1), ("B", 1)), onsite=((0, 0, 0.0), (1, 0, 0.0)), hops=tuple(hops),
                                 overlap=tuple(ovl), removable=("A", "B"))
    sc = hx.build_supercell(model.lattice_spec(), 10)
    with pytest.raises(hx.SolverError, match="not positive definite"):
        hx.solve_bands(model, sc, None, hx.make_bz_grid(model.lattice_spec(), 10, 1, "reduced"))


# ---- synchronisation safety of the flag-pipelined chases (compute-sanitizer is not available on this pool) -----
@pytest.mark.parametrize("opts", [{"HX_CHASE_RNW": 16}, {"HX_CHASE_RNW": 4}, {"HX_CHASE_RNW": 1},
                                  {"HX_CHASE_RNW": 16, "HX_CHASE_REG": 0}, {"HX_CHASE_RNW": 4, "HX_CHASE_REG": 0},
                                  {"HX_CHASE_RCL": 2}, {"HX_CHASE_RCL": 2, "HX_CHASE_REG": 0},
                                  {"HX_CHASE_REAL": 0}])
def test_chase_results_bitwise_repeatable(opts):
    """Every warp of a chase spins on its predecessor's progress counter before touching the band; a missing
    acquire/release would let a task read a tile before the previous sweep wrote it, which shows up as
    run-to-run differences.  The same batch is solved 12 times (with the GPU busy with a second batch on
    another context in between) and must give identical bits every time."""
    import threading

    model = hx.GrapheneNNModel()
    nu, q = (32, 1) if "HX_CHASE_RCL" in opts else (16, 2)
    sc = hx.build_supercell(model.lattice_spec(), nu)
    cell = hx.compile_cell(model, sc)
    kp = np.ascontiguousarray(hx.make_bz_grid(model.lattice_spec(), nu, q, "reduced").kpoints)
    words = sample_masks(sc.nunits, 0.05, 99, 1, 0, 8 if nu == 16 else 2)
    step = (HI_G - LO_G) / (NPTS - 1)
    other = _lib.Device.new_ctx(0, 0)
    noise = sample_masks(sc.nunits, 0.05, 5, 1, 0, 16)
    with _lib.options(**opts):
        ref, eigs0, _ = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01, want_eigs=True)
        for rep in range(12):
            th = threading.Thread(target=eval_batch, args=(cell, kp, noise, LO_G, step, NPTS, 0.01),
                                  kwargs={"ctx": other}) if rep % 3 == 0 else None
            if th:
                th.start()
            cur, eigs, _ = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01, want_eigs=True)
            if th:
                th.join()
            assert np.array_equal(cur, ref), rep
            assert np.array_equal(eigs, eigs0, equal_nan=True), rep


@pytest.mark.parametrize("opts", [{"HX_RU_BULK": 1, "HX_RU_TMA": 0}, {"HX_RU_TMA": 0}, {"HX_RU_TMA": 1}])
@pytest.mark.parametrize("nu,q", [(16, 2), (12, 1), (32, 1)])
def test_rank_update_variants(nu, q, opts):
    """The real rank update on the TMA engine (HX_RU_TMA=1, default: tensor-map boxes, 128-byte swizzle), the
    cp.async kernel and the per-column bulk-copy kernel, against the oracle."""
    check_batch("graphene", nu, q, 0.05, 4 if nu < 32 else 2, 13, (0, 1), opts=opts)


def test_c3_table_her2k_3m_option():
    """HX_HERK_3M=1: the 3M complex product in the Hermitian tier's her2k (1 CTA / SM) against zheevd."""
    check_batch("table", 8, 2, 0.05, 3, 2026, (0, 2), opts={"HX_HERK_3M": 1})


# ---- Gram path (G = C^T C, symmetric two-stage reduction) of the real IDOS-only batches ---------------------
@pytest.mark.parametrize("nu,q,count", [(16, 2, 8), (32, 1, 2), (12, 1, 6), (10, 2, 6), (20, 1, 3), (8, 2, 12)])
def test_gram_path_vs_svd_path_and_oracle(nu, q, count):
    """The IDOS of the Gram path (HX_GRAM=1: real batches whose zones avoid lambda = 0; off by default) equals the
    SVD path's (HX_GRAM=0) to rounding and the oracle (zhegv) within the north-star tolerance."""
    _, om, sc, cell, kp = _setup("graphene", nu, q)
    step = (HI_G - LO_G) / (NPTS - 1)
    words = sample_masks(sc.nunits, 0.05, 77, 2, 0, count)
    with _lib.options(HX_GRAM=1):
        gram, _, st1 = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
    with _lib.options(HX_GRAM=0):
        svd, _, st0 = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
    assert (st1 == 0).all() and (st0 == 0).all()
    np.testing.assert_allclose(gram, svd, rtol=0, atol=1e-11)
    ocell = O.make_cell(om, nu)
    for m in (0, count - 1):
        ref = O.solve_bands(ocell, om, words_to_int(words[m]), kp)
        rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), LO_G, HI_G, NPTS, 0.01, ocell.area)
        np.testing.assert_allclose(gram[m], rc, rtol=0, atol=IDOS_TOL)


def test_gram_path_high_vacancy_and_empty():
    """Many vacancies (zero modes, nA != nB) and an all-vacant mask through the Gram path."""
    _, om, sc, cell, kp = _setup("graphene", 16, 2)
    words = sample_masks(sc.nunits, 0.35, 5, 1, 0, 4)
    words[3] = np.uint64(0xFFFFFFFFFFFFFFFF)
    step = (HI_G - LO_G) / (NPTS - 1)
    with _lib.options(HX_GRAM=1):
        gram, _, st = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
    assert (st[:3] == 0).all() and (st[3] == _lib.HX_ST_EMPTY).all()
    assert np.all(gram[3] == 0.0)
    ocell = O.make_cell(om, 16)
    for m in range(3):
        ref = O.solve_bands(ocell, om, words_to_int(words[m]), kp)
        rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), LO_G, HI_G, NPTS, 0.01, ocell.area)
        np.testing.assert_allclose(gram[m], rc, rtol=0, atol=IDOS_TOL)


@pytest.mark.parametrize("opts", [{"HX_CHASE_RNW": 1}, {"HX_CHASE_RNW": 2}, {"HX_CHASE_RNW": 4}, {"HX_CHASE_RNW": 8},
                                  {"HX_CHASE_RNW": 16}, {"HX_CHASE_RCL": 2}, {"HX_CHASE_RCL": 4},
                                  {"HX_GRAM_CHASE": 0}, {"HX_GRAM_ASSEMBLE": 0}, {"HX_GRAM_WSPLIT": 0},
                                  {"HX_GRAM_SYM2": 0}, {"HX_GRAM_TRI": 0}])
@pytest.mark.parametrize("nu,q,count", [(16, 2, 6), (32, 1, 2), (14, 1, 4)])
def test_gram_chase_variants(nu, q, count, opts):
    """Every launch shape of the compact-band register-row symmetric chase (warps per matrix, cluster sizes), the
    dense-slab chase (HX_GRAM_CHASE=0), the dense-C Gram build (HX_GRAM_ASSEMBLE=0), the one-CTA W correction
    (HX_GRAM_WSPLIT=0) and the two-pass rank update (HX_GRAM_SYM2=0) against the oracle."""
    _, om, sc, cell, kp = _setup("graphene", nu, q)
    step = (HI_G - LO_G) / (NPTS - 1)
    words = sample_masks(sc.nunits, 0.07, 31, 1, 0, count)
    with _lib.options(HX_GRAM=1, **opts):
        gram, _, st = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
    assert (st == 0).all()
    ocell = O.make_cell(om, nu)
    for m in (0, count - 1):
        ref = O.solve_bands(ocell, om, words_to_int(words[m]), kp)
        rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), LO_G, HI_G, NPTS, 0.01, ocell.area)
        np.testing.assert_allclose(gram[m], rc, rtol=0, atol=IDOS_TOL)


# ---- Hermitian banded tier (tables): register-row chase on the compact complex band ---------------------------
@pytest.mark.parametrize("opts", [{"HX_HCHASE_RNW": 1}, {"HX_HCHASE_RNW": 2}, {"HX_HCHASE_RNW": 4},
                                  {"HX_HCHASE_RNW": 8}, {"HX_HCHASE_REG": 0}])
def test_hermitian_chase_variants(opts):
    """Every warps-per-matrix count of the register-row Hermitian chase (hx_chase.cuh: herm_chase_r_kernel) and the
    shared-memory-tile chase on the dense slab (HX_HCHASE_REG=0), 11-band table at nu = 6 (N = 396, defected so
    that d < N), eigenvalues and IDOS against zheevd."""
    check_batch("table", 6, 2, 0.08, 3, 7, (0, 2), opts=opts)


def test_hermitian_chase_bitwise_repeatable():
    """The flag-pipelined register-row Hermitian chase gives identical bits run after run (4 and 8 warps)."""
    _, om, sc, cell, kp = _setup("table", 6, 1)
    words = sample_masks(sc.nunits, 0.05, 3, 1, 0, 4)
    step = (HI_T - LO_T) / (NPTS - 1)
    for nw in (4, 8):
        with _lib.options(HX_HCHASE_RNW=nw):
            ref, eigs0, _ = eval_batch(cell, kp, words, LO_T, step, NPTS, 0.01, want_eigs=True)
            for _ in range(6):
                cur, eigs, _ = eval_batch(cell, kp, words, LO_T, step, NPTS, 0.01, want_eigs=True)
                assert np.array_equal(cur, ref) and np.array_equal(eigs, eigs0, equal_nan=True)


@pytest.mark.parametrize("opts", [{"HX_CHASE_RNW": 8}, {"HX_CHASE_RNW": 4}, {"HX_CHASE_RNW": 16}, {"HX_CHASE_RCL": 2},
                                  {"HX_CHASE_RCL": 4}])
def test_gram_chase_bitwise_repeatable(opts):
    """The flag-pipelined symmetric chase (half-task progress counters for the 8-warp and cluster launches) gives
    identical curves run after run, with a second batch running on another context in between."""
    import threading

    model = hx.GrapheneNNModel()
    nu, q = (32, 1) if "HX_CHASE_RCL" in opts else (16, 2)
    sc = hx.build_supercell(model.lattice_spec(), nu)
    cell = hx.compile_cell(model, sc)
    kp = np.ascontiguousarray(hx.make_bz_grid(model.lattice_spec(), nu, q, "reduced").kpoints)
    words = sample_masks(sc.nunits, 0.05, 99, 1, 0, 8 if nu == 16 else 2)
    step = (HI_G - LO_G) / (NPTS - 1)
    other = _lib.Device.new_ctx(0, 0)
    noise = sample_masks(sc.nunits, 0.05, 5, 1, 0, 16)
    with _lib.options(HX_GRAM=1, **opts):
        ref, _, _ = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
        for rep in range(12):
            th = threading.Thread(target=eval_batch, args=(cell, kp, noise, LO_G, step, NPTS, 0.01),
                                  kwargs={"ctx": other}) if rep % 3 == 0 else None
            if th:
                th.start()
            cur, _, _ = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
            if th:
                th.join()
            assert np.array_equal(cur, ref), rep


# ---- complex Gram path: G = C^H C through the Hermitian banded tier (non-time-reversal-invariant k-points) ------
@pytest.mark.parametrize("nu,q,count,p", [(12, 3, 4, 0.05), (16, 4, 3, 0.05), (10, 3, 6, 0.08), (24, 3, 2, 0.05),
                                          (14, 5, 3, 0.3)])
def test_complex_gram_path_vs_svd_path_and_oracle(nu, q, count, p):
    """IDOS-only batches with complex k-points (q >= 3) and N > 160: the default (HX_GRAM_C=1) forms G = C^H C and
    runs the Hermitian two-stage reduction; it equals the complex bidiagonal path (HX_GRAM_C=0) to rounding and the
    oracle (zhegv) within the north-star tolerance, also with many vacancies (nA != nB, zero modes)."""
    _, om, sc, cell, kp = _setup("graphene", nu, q)
    step = (HI_G - LO_G) / (NPTS - 1)
    words = sample_masks(sc.nunits, p, 41, 2, 0, count)
    with _lib.options(HX_GRAM_C=1):
        gram, _, st1 = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
    with _lib.options(HX_GRAM_C=0):
        svd, _, st0 = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
    assert (st1 == 0).all() and (st0 == 0).all()
    np.testing.assert_allclose(gram, svd, rtol=0, atol=1e-11)
    ocell = O.make_cell(om, nu)
    for m in (0, count - 1):
        ref = O.solve_bands(ocell, om, words_to_int(words[m]), kp)
        rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), LO_G, HI_G, NPTS, 0.01, ocell.area)
        np.testing.assert_allclose(gram[m], rc, rtol=0, atol=IDOS_TOL)


def test_complex_gram_path_all_vacant_and_repeatable():
    _, om, sc, cell, kp = _setup("graphene", 12, 3)
    step = (HI_G - LO_G) / (NPTS - 1)
    words = sample_masks(sc.nunits, 0.05, 8, 1, 0, 3)
    words[2] = np.uint64(0xFFFFFFFFFFFFFFFF)
    with _lib.options(HX_GRAM_C=1):
        a, _, st = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
        b, _, _ = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
    assert (st[:2] == 0).all() and (st[2] == _lib.HX_ST_EMPTY).all()
    assert np.all(a[2] == 0.0) and np.array_equal(a, b)


# ---- Gram path of the shared-memory tier (S in (32, 64]: G = C^H C in registers, hx_smallgram.cuh) ----------
@pytest.mark.parametrize("nu,q,conc,count", [(8, 4, 0.05, 40), (8, 3, 0.05, 24), (8, 2, 0.05, 24), (7, 5, 0.1, 16),
                                             (6, 3, 0.1, 16), (5, 4, 0.05, 16), (8, 4, 0.3, 24), (7, 2, 0.25, 16)])
def test_small_gram_path_vs_golub_kahan_and_oracle(nu, q, conc, count):
    """N = 50..128 tiers (c2's N = 128 tier is nu = 8, q = 4): the register-resident Hermitian tridiagonalisation of
    G = C^H C (complex k-points) / C^T C (TRIM k-points) with the mu = sigma^2 zone path (HX_SMALL_GRAM=1, default
    for IDOS-only calls) equals the Golub-Kahan path (HX_SMALL_GRAM=0) to rounding and the oracle within the
    north-star tolerance; rectangular / padded blocks at high vacancy counts."""
    _, om, sc, cell, kp = _setup("graphene", nu, q)
    step = (HI_G - LO_G) / (NPTS - 1)
    words = sample_masks(sc.nunits, conc, 91, 2, 0, count)
    with _lib.options(HX_SMALL_GRAM=1):
        gram, _, st1 = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
        again, _, _ = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
    with _lib.options(HX_SMALL_GRAM=0):
        gk, _, st0 = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
    assert (st1 == 0).all() and (st0 == 0).all()
    assert np.array_equal(gram, again)
    np.testing.assert_allclose(gram, gk, rtol=0, atol=1e-11)
    ocell = O.make_cell(om, nu)
    for m in (0, count // 2, count - 1):
        ref = O.solve_bands(ocell, om, words_to_int(words[m]), kp)
        rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), LO_G, HI_G, NPTS, 0.01, ocell.area)
        np.testing.assert_allclose(gram[m], rc, rtol=0, atol=IDOS_TOL)


def test_small_gram_path_all_vacant_and_single_site():
    """All-vacant mask (zero curve, HX_ST_EMPTY), a mask that keeps one unit only, and a pristine cell through the
    small-tier Gram path."""
    _, om, sc, cell, kp = _setup("graphene", 8, 4)
    words = sample_masks(sc.nunits, 0.05, 3, 1, 0, 4)
    words[1] = np.uint64(0xFFFFFFFFFFFFFFFF)
    words[2] = np.uint64(0xFFFFFFFFFFFFFFFF)
    words[2, 0] = np.uint64(0xFFFFFFFFFFFFFFFE)
    words[3] = np.uint64(0)
    step = (HI_G - LO_G) / (NPTS - 1)
    with _lib.options(HX_SMALL_GRAM=1):
        gram, _, st = eval_batch(cell, kp, words, LO_G, step, NPTS, 0.01)
    assert (st[1] == _lib.HX_ST_EMPTY).all() and np.all(gram[1] == 0.0)
    assert (st[[0, 2, 3]] == 0).all()
    ocell = O.make_cell(om, 8)
    for m in (0, 2, 3):
        ref = O.solve_bands(ocell, om, words_to_int(words[m]), kp)
        rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), LO_G, HI_G, NPTS, 0.01, ocell.area)
        np.testing.assert_allclose(gram[m], rc, rtol=0, atol=IDOS_TOL)


# ---- zone path of the eigenvalue stage: fused per-matrix refinement / staged multisection vs the item list ----
@pytest.mark.parametrize("kind,nu,q,count", [("graphene", 16, 2, 12), ("graphene", 32, 1, 3), ("graphene", 8, 4, 24),
                                             ("graphene", 11, 1, 6), ("graphene", 12, 3, 4), ("table", 4, 2, 6),
                                             ("table", 6, 1, 3), ("graphene", 23, 1, 2), ("table", 10, 1, 2),
                                             ("graphene", 24, 3, 2)])
def test_zone_refinement_variants_same_bits(kind, nu, q, count):
    """The refinement fused into the zone-count kernel (HX_ZONE_FUSE, matrices below 1024) and the staged
    multisection on the grouped item list (HX_ZONE_STAGE, Gram tridiagonals from S = 1024) run the same searches
    with the same arguments as the global item list: curves bitwise equal; Gram (S = 256, 1024, 64), TGK (odd S,
    complex k) and Hermitian (table) tridiagonals, below and above the multisection threshold (N = 1024)."""
    _, om, sc, cell, kp = _setup(kind, nu, q)
    lo, hi = (LO_T, HI_T) if kind == "table" else (LO_G, HI_G)
    step = (hi - lo) / (NPTS - 1)
    words = sample_masks(sc.nunits, 0.06, 57, 1, 0, count)
    base, _, st = eval_batch(cell, kp, words, lo, step, NPTS, 0.01)
    assert (st == 0).all()
    for opts in ({"HX_ZONE_FUSE": 0}, {"HX_ZONE_STAGE": 0}, {"HX_ZONE_FUSE": 0, "HX_ZONE_STAGE": 0}):
        with _lib.options(**opts):
            alt, _, st2 = eval_batch(cell, kp, words, lo, step, NPTS, 0.01)
        assert (st2 == 0).all()
        assert np.array_equal(base, alt), opts
    # the G-lane multisection (the method of matrices too large to stage): staged and unstaged give the same bits,
    # and the per-thread Newton search agrees with it to the refinement tolerance
    lanes = {"HX_GRAM_REFINE_LANES": 8, "HX_REFINE_LANES": 4}
    with _lib.options(**lanes):
        ms, _, st3 = eval_batch(cell, kp, words, lo, step, NPTS, 0.01)
    with _lib.options(HX_ZONE_STAGE=0, **lanes):
        ms0, _, st4 = eval_batch(cell, kp, words, lo, step, NPTS, 0.01)
    assert (st3 == 0).all() and (st4 == 0).all()
    assert np.array_equal(ms, ms0)
    np.testing.assert_allclose(ms, base, rtol=0, atol=1e-11)
    ocell = O.make_cell(om, nu)
    ref = O.solve_bands(ocell, om, words_to_int(words[0]), kp)
    rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), lo, hi, NPTS, 0.01, ocell.area)
    np.testing.assert_allclose(base[0], rc, rtol=0, atol=IDOS_TOL)
