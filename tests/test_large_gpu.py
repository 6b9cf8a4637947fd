"""Config-4 scale (nu = 64, N = 8192) through the bipartite banded tier, checked with size-independent
properties: band folding of the unperturbed supercell at Gamma (analytic two-band dispersion on the
64 x 64 folded fundamental grid, tests/test_spectrum.py:94-110 style) and the IDOS plateau
(= surviving orbitals / area, tests/test_qoi.py:83-92 style) for a defected sample."""

import numpy as np
import pytest

import paper_1611_09784_b200 as hx
from paper_1611_09784_b200.sampling import sample_masks
from paper_1611_09784_b200.solver import eval_batch

pytestmark = pytest.mark.gpu

LO, HI, NPTS = -6.580201874549387, 14.863393148450246, 201


def analytic_bands(model, kpts):
    spec = model.lattice_spec()
    a1, a2 = np.asarray(spec.a1), np.asarray(spec.a2)
    w = np.abs(1.0 + np.exp(-1j * kpts @ a1) + np.exp(-1j * kpts @ a2))
    lo = (model.eps_2p + model.t * w) / (1.0 + model.s * w)
    hi = (model.eps_2p - model.t * w) / (1.0 - model.s * w)
    return np.sort(np.concatenate([lo, hi]))


@pytest.mark.parametrize("nu", [24, 64])
def test_unperturbed_gamma_folds_fundamental_bands(nu):
    model = hx.GrapheneNNModel()
    spec = model.lattice_spec()
    sc = hx.build_supercell(spec, nu)
    cell = hx.compile_cell(model, sc)
    words = np.zeros((1, max(1, (sc.nunits + 63) // 64)), dtype=np.uint64)
    _, eigs, status = eval_batch(cell, np.zeros((1, 2)), words, LO, (HI - LO) / (NPTS - 1), NPTS, 0.01,
                                 want_eigs=True)
    assert (status == 0).all()
    b1, b2 = spec.reciprocal_vectors()
    ii, jj = np.meshgrid(np.arange(nu), np.arange(nu), indexing="ij")
    kf = (ii.reshape(-1, 1) * b1 + jj.reshape(-1, 1) * b2) / nu
    ref = analytic_bands(model, kf)
    assert np.max(np.abs(eigs[0, 0] - ref)) <= 1e-10 * (ref.max() - ref.min())


def test_nu64_defected_sample_plateau_and_monotone():
    model = hx.GrapheneNNModel()
    sc = hx.build_supercell(model.lattice_spec(), 64)
    cell = hx.compile_cell(model, sc)
    words = sample_masks(sc.nunits, 0.02, 2026, 1, 0, 1)
    vac = sum(bin(int(w)).count("1") for w in words[0])
    kp = hx.make_bz_grid(model.lattice_spec(), 64, 2, "reduced").kpoints  # Gamma + 3 points (config 4)
    curves, _, status = eval_batch(cell, kp, words, LO, (HI - LO) / (NPTS - 1), NPTS, 0.01)
    assert (status == 0).all()
    d = sc.nunits - vac
    assert curves[0, -1] == pytest.approx(d / sc.area, abs=1e-12)
    assert np.all(np.diff(curves[0]) >= -1e-12)


def test_nu46_defected_matches_oracle_on_the_large_real_path():
    """S = 46^2 = 2116 >= 2048: the real-storage stage 1 with the fused schedule (trailing updates applied
    by the next xv pass) and the clustered real chase (several SMs per matrix) - a defected sample at Gamma
    against the oracle (LAPACK zhegv on the N = 4232 pencil, ~10 s on the host): eigenvalues within
    1e-10 x width, IDOS within 1e-9."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    import hexmc_oracle as O

    nu = 46
    model = hx.GrapheneNNModel()
    spec = model.lattice_spec()
    sc = hx.build_supercell(spec, nu)
    cell = hx.compile_cell(model, sc)
    kp = hx.make_bz_grid(spec, nu, 1, "reduced").kpoints
    words = sample_masks(sc.nunits, 0.02, 5, 2, 0, 1)
    curves, eigs, status = eval_batch(cell, kp, words, LO, (HI - LO) / (NPTS - 1), NPTS, 0.01, want_eigs=True)
    assert (status == 0).all()
    om = O.graphene_model()
    ocell = O.make_cell(om, nu)
    key = sum(int(w) << (64 * i) for i, w in enumerate(words[0]))
    ref = O.solve_bands(ocell, om, key, kp)
    d = ref.shape[1]
    assert np.max(np.abs(eigs[0, :, :d] - ref)) <= 1e-10 * (ref.max() - ref.min())
    rc = O.idos_from_bands(ref, np.full(len(kp), 1.0 / len(kp)), LO, HI, NPTS, 0.01, ocell.area)
    np.testing.assert_allclose(curves[0], rc, rtol=0, atol=1e-9)
    # the IDOS-only call takes the Gram path (G = C^T C, lower-tile rank-2k update, 4-SM clustered symmetric chase
    # with release / acquire half-task counters, 8-lane multisection in mu = sigma^2): same oracle, same tolerance
    fast, _, st = eval_batch(cell, kp, words, LO, (HI - LO) / (NPTS - 1), NPTS, 0.01)
    assert (st == 0).all()
    np.testing.assert_allclose(fast[0], rc, rtol=0, atol=1e-9)
