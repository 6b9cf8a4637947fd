"""GPU parity: the CUDA path (through the C-ABI) against the reference-generated goldens and the oracle.

Tolerances (BASELINE.json north_star): eigenvalues <= 1e-10 x spectral width; per-sample IDOS <= 1e-9;
level means <= 1e-9; sharp counts identical except within 1e-10 of a grid energy; masks bit-identical.
"""

import numpy as np
import pytest

import hexmc_oracle as O
from conftest import TABLE, golden, words_to_int

import paper_1611_09784_b200 as hx
from paper_1611_09784_b200.solver import eval_batch

pytestmark = pytest.mark.gpu

EIG_TOL = 1e-10  # x spectral width
IDOS_TOL = 1e-9


def model_of(name):
    return hx.load_coupling_table(TABLE) if name.startswith("t") else hx.GrapheneNNModel()


@pytest.mark.parametrize("name,table,nu", [
    ("g2_v3", False, 2), ("g1_gamma", False, 1), ("g4_rand", False, 4), ("g3_none", False, 3),
    ("t2_v1", True, 2), ("t1_none", True, 1)])
def test_device_assembly_matches_reference(name, table, nu):
    g = golden("assembly.npz")
    model = hx.load_coupling_table(TABLE) if table else hx.GrapheneNNModel()
    sc = hx.build_supercell(model.lattice_spec(), nu)
    cfg = hx.DefectConfiguration.from_key(sc, words_to_int(g[f"{name}_mask"]))
    pair = hx.assemble_bloch(model, sc, cfg, g[f"{name}_k"])
    np.testing.assert_allclose(pair.H, g[f"{name}_H"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(pair.S, g[f"{name}_S"], rtol=0, atol=1e-13)


@pytest.mark.parametrize("name", ["g4q6", "g8q4", "g16q1", "t2q4", "t4q2"])
def test_eigenvalues_and_curves_match_reference(name):
    g = golden("eigs_curves.npz")
    model = model_of(name)
    nu, q = (int(x) for x in g[f"{name}_meta"])
    lo, hi, npts = g[f"{name}_grid"]
    npts = int(npts)
    sc = hx.build_supercell(model.lattice_spec(), nu)
    cell = hx.compile_cell(model, sc)
    kp = g[f"{name}_kpoints"]
    words = g[f"{name}_masks"]
    step = (hi - lo) / (npts - 1)
    curves, eigs, status = eval_batch(cell, kp, words, lo, step, npts, 0.01, want_eigs=True)
    assert (status == 0).all()
    ref = g[f"{name}_eigs"]
    width = np.nanmax(ref) - np.nanmin(ref)
    np.testing.assert_array_equal(np.isnan(eigs), np.isnan(ref))
    assert np.nanmax(np.abs(eigs - ref)) <= EIG_TOL * width
    np.testing.assert_allclose(curves, g[f"{name}_curves"], rtol=0, atol=IDOS_TOL)
    np.testing.assert_allclose(curves, g[f"{name}_curves_full"], rtol=0, atol=IDOS_TOL)
    # without the eigenvalue output the IDOS takes the fast paths (zone counts + Newton for N >= 96,
    # early-settling bisection below): same curves
    fast, _, status = eval_batch(cell, kp, words, lo, step, npts, 0.01)
    assert (status == 0).all()
    np.testing.assert_allclose(fast, g[f"{name}_curves"], rtol=0, atol=IDOS_TOL)
    sharp, _, _ = eval_batch(cell, kp, words, lo, step, npts, 0.01, sharp=True)
    ref_sharp = g[f"{name}_sharp"]
    diff = np.abs(sharp - ref_sharp) > 1e-12
    if diff.any():
        # only allowed where an eigenvalue sits within 1e-10 of a grid energy
        grid = lo + step * np.arange(npts)
        for m, j in zip(*np.nonzero(diff)):
            e = ref[m][~np.isnan(ref[m])]
            assert np.min(np.abs(e - grid[j])) < 1e-10


def test_solve_bands_gamma_and_analytic():
    model = hx.GrapheneNNModel()
    sc = hx.build_supercell(model.lattice_spec(), 1)
    grid = hx.make_bz_grid(model.lattice_spec(), 1, 1, "reduced")
    bands = hx.solve_bands(model, sc, None, grid)
    np.testing.assert_allclose(bands.energies[0], [3 * model.t / (1 + 3 * model.s), -3 * model.t / (1 - 3 * model.s)],
                               rtol=0, atol=1e-12)
    assert bands.energies[0][0] == pytest.approx(-6.5602, abs=1e-4)
    assert bands.energies[0][1] == pytest.approx(14.8434, abs=1e-4)


def test_band_folding_nu2_vs_nu1():
    model = hx.GrapheneNNModel()
    spec = model.lattice_spec()
    b1 = hx.solve_bands(model, hx.build_supercell(spec, 1), None, hx.make_bz_grid(spec, 1, 8, "reduced"))
    b2 = hx.solve_bands(model, hx.build_supercell(spec, 2), None, hx.make_bz_grid(spec, 2, 4, "reduced"))
    np.testing.assert_allclose(np.sort(b2.energies.reshape(-1)), np.sort(b1.energies.reshape(-1)), atol=1e-9)


def test_non_pd_overlap_raises_solver_error():
    entries = []
    for di, dj in ((0, 0), (-1, 0), (0, -1)):
        entries.append((di, dj, 0, 0, 1, 0, 0.5 + 0j))
        entries.append((-di, -dj, 1, 0, 0, 0, 0.5 + 0j))
    model = hx.MultiOrbitalModel(orbitals=(("A", 1), ("B", 1)), onsite=((0, 0, 0.0), (1, 0, 0.0)),
                                 hops=((0, 0, 0, 0, 1, 0, -1.0 + 0j), (0, 0, 1, 0, 0, 0, -1.0 + 0j)),
                                 overlap=tuple(entries), removable=("A", "B"))
    sc = hx.build_supercell(model.lattice_spec(), 1)
    grid = hx.make_bz_grid(model.lattice_spec(), 1, 1, "reduced")
    with pytest.raises(hx.SolverError, match=r"k=\("):
        hx.solve_bands(model, sc, None, grid)


def test_general_pencil_matches_zhegv():
    # a PD overlap table: graphene as a general table (overlap couplings) -> Cholesky path
    entries, hops = [], []
    for di, dj in ((0, 0), (-1, 0), (0, -1)):
        entries += [(di, dj, 0, 0, 1, 0, 0.129 + 0j), (-di, -dj, 1, 0, 0, 0, 0.129 + 0j)]
        hops += [(di, dj, 0, 0, 1, 0, -3.033 + 0j), (-di, -dj, 1, 0, 0, 0, -3.033 + 0j)]
    model = hx.MultiOrbitalModel(orbitals=(("A", 1), ("B", 1)), onsite=((0, 0, 0.0), (1, 0, 0.0)),
                                 hops=tuple(hops), overlap=tuple(entries), removable=("A", "B"))
    spec = model.lattice_spec()
    sc = hx.build_supercell(spec, 3)
    cfg = hx.sample_defects(sc, 0.2, hx.SeedSpec(5, 1, 2))
    grid = hx.make_bz_grid(spec, 3, 2, "reduced")
    bands = hx.solve_bands(model, sc, cfg, grid)
    om = O.graphene_model()
    ocell = O.make_cell(om, 3)
    ref = O.solve_bands(ocell, om, cfg.key, grid.kpoints)
    assert np.max(np.abs(bands.energies - ref)) <= EIG_TOL * (ref.max() - ref.min())


def test_curves_independent_of_batch_composition():
    model = hx.GrapheneNNModel()
    sc = hx.build_supercell(model.lattice_spec(), 4)
    cell = hx.compile_cell(model, sc)
    kp = hx.make_bz_grid(model.lattice_spec(), 4, 6, "reduced").kpoints
    from paper_1611_09784_b200.sampling import sample_masks

    w = sample_masks(sc.nunits, 0.05, 2026, 1, 0, 64)
    a, _, _ = eval_batch(cell, kp, w, -6.58, 0.107, 201, 0.01)
    perm = np.random.default_rng(0).permutation(64)
    b, _, _ = eval_batch(cell, kp, w[perm], -6.58, 0.107, 201, 0.01)
    c, _, _ = eval_batch(cell, kp, w[:7], -6.58, 0.107, 201, 0.01)
    assert np.array_equal(a[perm], b)
    assert np.array_equal(a[:7], c)


def test_engine_levels_match_reference():
    g = golden("levels.npz")
    eng = hx.Engine(hx.GrapheneNNModel(), nq=16, delta=0.01, master_seed=2026, bz_mode="reduced", energy_points=201)
    assert (eng.grid.lo, eng.grid.hi) == pytest.approx((g["grid"][0], g["grid"][1]), abs=1e-13)
    recs = g["records"]
    for level, (n, M) in enumerate(((4, 24), (8, 8)), start=1):
        s = eng.sample_level(level, n, M, 0.05, with_cv=level > 1)
        np.testing.assert_allclose(s.full, g[f"L{level}_full"], rtol=0, atol=IDOS_TOL)
        np.testing.assert_allclose(s.stats.mean, g[f"L{level}_mean"], rtol=0, atol=IDOS_TOL)
        np.testing.assert_allclose(s.stats.sample_variance, g[f"L{level}_var"], rtol=0, atol=IDOS_TOL)
        assert s.stats.cache_hits == recs[level - 1][4]
    t = hx.load_coupling_table(TABLE)
    et = hx.Engine(t, nq=4, delta=0.01, master_seed=2026, bz_mode="reduced", energy_points=201,
                   energy_range=(-2.932, 4.740))
    s = et.sample_level(1, 2, 6, 0.05, with_cv=False)
    np.testing.assert_allclose(s.full, g["table_L1_full"], rtol=0, atol=IDOS_TOL)
    np.testing.assert_allclose(s.stats.mean, g["table_L1_mean"], rtol=0, atol=IDOS_TOL)


def test_all_vacant_gives_zero_curve_and_plateau():
    eng = hx.Engine(hx.GrapheneNNModel(), nq=8, delta=0.02, master_seed=99, energy_points=512)
    s = eng.sample_level(1, 1, 3, p_vac=1.0, with_cv=False)
    assert np.array_equal(s.full, np.zeros_like(s.full))
    plan = hx.LevelPlan(ns=(2, 4), samples=(6, 3), nq=8, p_vac=0.0, delta=0.02)
    _, sets = eng.run_mlmc(plan)
    for sset in sets:
        n = sset.stats.n
        assert np.allclose(sset.full[:, -1], 2.0 * n * n / eng.supercell(n).area, atol=1e-9)


@pytest.mark.parametrize("nu,q,p", [(10, 2, 0.2), (11, 1, 0.3), (12, 1, 0.05), (16, 2, 0.1), (12, 1, 0.5),
                                    (13, 1, 0.4), (14, 1, 0.45), (17, 1, 0.35), (20, 2, 0.05), (24, 1, 0.1)])
def test_bipartite_banded_tier_matches_oracle(nu, q, p):
    """graphene N = 2nu^2 > 160 goes through the bipartite banded tier (nA != nB after vacancies).  High
    vacancy rates leave exactly-zero rows/columns whose reflections produce ever smaller noise columns
    (down to the denormal range): the reflectors must stay unitary (HX_REFLECTOR_TINY).  Even nu with
    q <= 2 (S = nu^2 % 4 == 0, real batch) run the real-storage stage 1 (hx_real.cuh: one-CTA 512-row
    panels at nu = 20, two-CTA clusters at nu = 24); odd nu the complex-storage one."""
    model = hx.GrapheneNNModel()
    spec = model.lattice_spec()
    sc = hx.build_supercell(spec, nu)
    cell = hx.compile_cell(model, sc)
    kp = hx.make_bz_grid(spec, nu, q, "reduced").kpoints
    from paper_1611_09784_b200.sampling import sample_masks

    words = sample_masks(sc.nunits, p, 77, 3, 0, 3)
    lo, hi, npts = -6.580201874549387, 14.863393148450246, 201
    curves, eigs, status = eval_batch(cell, kp, words, lo, (hi - lo) / (npts - 1), npts, 0.01, want_eigs=True)
    assert (status == 0).all()
    om = O.graphene_model()
    ocell = O.make_cell(om, nu)
    for m in range(len(words)):
        ref = O.solve_bands(ocell, om, words_to_int(words[m]), kp)
        d = ref.shape[1]
        assert np.all(np.isnan(eigs[m, :, d:]))
        assert np.max(np.abs(eigs[m, :, :d] - ref)) <= EIG_TOL * (ref.max() - ref.min())
        rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), lo, hi, npts, 0.01, ocell.area)
        np.testing.assert_allclose(curves[m], rc, rtol=0, atol=IDOS_TOL)


@pytest.mark.parametrize("kind,nu,q,p", [("table", 4, 2, 0.4), ("table", 5, 1, 0.5), ("graphene", 8, 2, 0.5),
                                         ("graphene", 4, 3, 0.6), ("graphene", 6, 2, 0.45)])
def test_high_vacancy_tiers_match_oracle(kind, nu, q, p):
    """Every tier at high vacancy rates (exact zero rows/columns -> noise-only reflector columns): the
    Hermitian banded tier (table nu >= 4), the shared-memory bidiagonalisation (CTA: S = 64, warp: S <= 32)."""
    model = hx.load_coupling_table(TABLE) if kind == "table" else hx.GrapheneNNModel()
    om = O.parse_table(str(TABLE)) if kind == "table" else O.graphene_model()
    spec = model.lattice_spec()
    sc = hx.build_supercell(spec, nu)
    cell = hx.compile_cell(model, sc)
    kp = hx.make_bz_grid(spec, nu, q, "reduced").kpoints
    from paper_1611_09784_b200.sampling import sample_masks

    words = sample_masks(sc.nunits, p, 91, 2, 0, 3)
    lo, hi, npts = (-2.952, 4.760, 201) if kind == "table" else (-6.580201874549387, 14.863393148450246, 201)
    curves, eigs, status = eval_batch(cell, kp, words, lo, (hi - lo) / (npts - 1), npts, 0.01, want_eigs=True)
    assert (status == 0).all()
    ocell = O.make_cell(om, nu)
    for m in range(len(words)):
        ref = O.solve_bands(ocell, om, words_to_int(words[m]), kp)
        d = ref.shape[1]
        assert np.max(np.abs(eigs[m, :, :d] - ref)) <= EIG_TOL * (ref.max() - ref.min())
        rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), lo, hi, npts, 0.01, ocell.area)
        np.testing.assert_allclose(curves[m], rc, rtol=0, atol=IDOS_TOL)


def test_run_mlmc_batched_equals_level_by_level():
    """run_mlmc submits every level at once; means, variances and cache hits must equal sampling the levels
    one after another (cross-level hits: level l's quarters at nu/2 meet level l-1's parents)."""
    kw = dict(nq=16, delta=0.01, master_seed=2026, bz_mode="reduced", energy_points=201)
    plan = hx.LevelPlan(ns=(2, 4, 8), samples=(64, 16, 4), nq=16, p_vac=0.1, delta=0.01)
    a = hx.Engine(hx.GrapheneNNModel(), **kw)
    _, sets = a.run_mlmc(plan)
    b = hx.Engine(hx.GrapheneNNModel(), **kw)
    for idx, (n, m) in enumerate(zip(plan.ns, plan.samples), start=1):
        s = b.sample_level(idx, n, m, plan.p_vac, with_cv=idx > 1)
        t = sets[idx - 1]
        assert np.array_equal(s.full, t.full)
        assert np.array_equal(s.stats.mean, t.stats.mean)
        assert s.stats.cache_hits == t.stats.cache_hits


def test_exhaustive_matches_oracle_enumeration():
    """run_exhaustive (runner.py:380-415): binomially weighted mean over all 2^N outcomes; nu = 1, p = 0.5 has
    terminal value 1.0 (the reference's test_cli.py:109-120), and the whole curve equals the oracle's own
    enumeration."""
    lo, hi, npts = -6.580201874549387, 14.863393148450246, 201
    eng = hx.Engine(hx.GrapheneNNModel(), nq=6, delta=0.01, master_seed=1, bz_mode="reduced", energy_points=npts,
                    energy_range=(lo + 0.02, hi - 0.02))
    res = eng.run_exhaustive(1, 0.5)
    assert res.nconfigs == 4 and res.weight_sum == pytest.approx(1.0, abs=1e-15)
    assert res.mean[-1] == pytest.approx(1.0, abs=1e-12)
    om = O.graphene_model()
    cell = O.make_cell(om, 1)
    kp = hx.make_bz_grid(hx.GrapheneNNModel().lattice_spec(), 1, 6, "reduced").kpoints
    w = np.full(len(kp), 1.0 / len(kp))
    want = np.zeros(npts)
    for mask in range(4):
        nvac = bin(mask).count("1")
        weight = 0.5 ** nvac * 0.5 ** (2 - nvac)
        if nvac == 2:
            continue  # all removed: zero curve
        bands = O.solve_bands(cell, om, mask, kp)
        want += weight * O.idos_from_bands(bands, w, lo, hi, npts, 0.01, cell.area)
    np.testing.assert_allclose(res.mean, want, rtol=0, atol=IDOS_TOL)


def test_empty_and_mixed_batches_on_the_zone_path():
    """nmasks = 0 is a no-op; a zone-path batch (N = 128) mixing the pristine, a fully vacant and random
    masks gives each mask the curve it gets alone (no cross-talk through the fixed-point accumulators)."""
    model = hx.GrapheneNNModel()
    sc = hx.build_supercell(model.lattice_spec(), 8)
    cell = hx.compile_cell(model, sc)
    kp = hx.make_bz_grid(model.lattice_spec(), 8, 2, "reduced").kpoints
    lo, hi, npts = -6.580201874549387, 14.863393148450246, 201
    step = (hi - lo) / (npts - 1)
    curves, _, status = eval_batch(cell, kp, np.zeros((0, 2), dtype=np.uint64), lo, step, npts, 0.01)
    assert curves.shape == (0, npts) and status.shape == (0, len(kp))
    from paper_1611_09784_b200.sampling import sample_masks

    words = np.concatenate([np.zeros((1, 2), np.uint64), np.full((1, 2), np.iinfo(np.uint64).max, np.uint64),
                            sample_masks(sc.nunits, 0.1, 5, 1, 0, 6)])
    both, _, status = eval_batch(cell, kp, words, lo, step, npts, 0.01)
    assert (status[1] == 3).all() and (status[[0, 2, 3]] == 0).all()
    assert np.array_equal(both[1], np.zeros(npts))
    for i in (0, 3, 7):
        alone, _, _ = eval_batch(cell, kp, words[i:i + 1], lo, step, npts, 0.01)
        np.testing.assert_array_equal(both[i], alone[0])
    om = O.graphene_model()
    ocell = O.make_cell(om, 8)
    ref = O.idos_from_bands(O.solve_bands(ocell, om, 0, kp), np.full(len(kp), 1.0 / len(kp)), lo, hi, npts, 0.01,
                            ocell.area)
    np.testing.assert_allclose(both[0], ref, rtol=0, atol=IDOS_TOL)


@pytest.mark.parametrize("nu,q", [(4, 8), (8, 4), (4, 6), (3, 5)])
def test_time_reversal_pairs_give_the_same_curves(nu, q, monkeypatch):
    """Graphene (real amplitudes): merging k and -k (multiplicity 2, hx_eval_idos_batch_k) reproduces the
    curves of the full reference grid, and the oracle's."""
    from paper_1611_09784_b200.sampling import sample_masks
    from paper_1611_09784_b200.solver import time_reversal_reduce

    model = hx.GrapheneNNModel()
    sc = hx.build_supercell(model.lattice_spec(), nu)
    cell = hx.compile_cell(model, sc)
    assert cell.time_reversal_symmetric
    kp = hx.make_bz_grid(model.lattice_spec(), nu, q, "reduced").kpoints
    reps, mult = time_reversal_reduce(model.lattice_spec(), nu, kp)
    lo, hi, npts = -6.580201874549387, 14.863393148450246, 201
    step = (hi - lo) / (npts - 1)
    words = sample_masks(sc.nunits, 0.1, 11, 1, 0, 12)
    full, _, st1 = eval_batch(cell, kp, words, lo, step, npts, 0.01)
    paired, _, st2 = eval_batch(cell, reps, words, lo, step, npts, 0.01, kmult=mult)
    assert (st1 == 0).all() and (st2 == 0).all() and st2.shape == (12, len(reps))
    np.testing.assert_allclose(paired, full, rtol=0, atol=1e-11)
    om = O.graphene_model()
    ocell = O.make_cell(om, nu)
    key = sum(int(w) << (64 * i) for i, w in enumerate(words[3]))
    ref = O.idos_from_bands(O.solve_bands(ocell, om, key, kp), np.full(len(kp), 1.0 / len(kp)), lo, hi, npts, 0.01,
                            ocell.area)
    np.testing.assert_allclose(paired[3], ref, rtol=0, atol=IDOS_TOL)
    # the Engine uses the paired sets; switching them off gives the same level curves
    eng = hx.Engine(model, nq=nu * q, delta=0.01, master_seed=4, bz_mode="reduced", energy_points=npts,
                    energy_range=(lo + 0.02, hi - 0.02))
    a = eng.sample_level(1, nu, 8, 0.1, with_cv=False).full
    monkeypatch.setenv("HX_NO_TIME_REVERSAL", "1")
    eng2 = hx.Engine(model, nq=nu * q, delta=0.01, master_seed=4, bz_mode="reduced", energy_points=npts,
                     energy_range=(lo + 0.02, hi - 0.02))
    b = eng2.sample_level(1, nu, 8, 0.1, with_cv=False).full
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-11)
