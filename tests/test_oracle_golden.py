"""Pin the CPU oracle against fixtures produced by the reference itself (oracle/make_golden.py)."""

import json

import numpy as np
import pytest

import hexmc_oracle as O
from conftest import TABLE, golden, words_to_int

LO_G, HI_G = -6.580201874549387, 14.863393148450246


def test_rng_numpy_and_pure_python_match_reference_draws():
    g = golden("rng.npz")
    streams, draws = g["streams"], g["draws"]
    for idx in range(0, len(streams), 7):
        s, lv, r = (int(x) for x in streams[idx])
        np.testing.assert_array_equal(O.numpy_uniforms(s, lv, r, 16), draws[idx])
        np.testing.assert_array_equal(O.seedseq_pcg64_uniforms(s, lv, r, 16), draws[idx])


@pytest.mark.parametrize("nu", [1, 2, 4, 8, 16, 32])
def test_masks_bit_identical(nu):
    g = golden("rng.npz")
    words = g[f"graphene_nu{nu}"]
    nunits = 2 * nu * nu
    for m in range(len(words)):
        assert O.sample_mask(nunits, 0.05, 2026, 1 + (nu % 5), m) == words_to_int(words[m])


@pytest.mark.parametrize("name,table,nu", [
    ("g2_v3", False, 2), ("g1_gamma", False, 1), ("g4_rand", False, 4), ("g3_none", False, 3),
    ("t2_v1", True, 2), ("t1_none", True, 1)])
def test_assembly_matches_reference(name, table, nu):
    g = golden("assembly.npz")
    model = O.parse_table(TABLE) if table else O.graphene_model()
    cell = O.make_cell(model, nu)
    H, S = O.assemble(cell, model, words_to_int(g[f"{name}_mask"]), g[f"{name}_k"])
    np.testing.assert_allclose(H, g[f"{name}_H"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(S, g[f"{name}_S"], rtol=0, atol=1e-14)


@pytest.mark.parametrize("name", ["g4q6", "g8q4", "t2q4", "t4q2"])
def test_eigs_and_curves_match_reference(name):
    g = golden("eigs_curves.npz")
    model = O.parse_table(TABLE) if name.startswith("t") else O.graphene_model()
    nu, q = (int(x) for x in g[f"{name}_meta"])
    lo, hi, npts = g[f"{name}_grid"]
    npts = int(npts)
    cell = O.make_cell(model, nu)
    kp, kw = O.bz_grid(nu, q, "reduced")
    np.testing.assert_array_equal(kp, g[f"{name}_kpoints"])
    for m in range(min(3, len(g[f"{name}_masks"]))):
        mask = words_to_int(g[f"{name}_masks"][m])
        bands = O.solve_bands(cell, model, mask, kp)
        ref = g[f"{name}_eigs"][m][:, : bands.shape[1]]
        np.testing.assert_allclose(bands, ref, rtol=0, atol=1e-12)
        curve = O.idos_from_bands(bands, kw, lo, hi, npts, 0.01, cell.area)
        np.testing.assert_allclose(curve, g[f"{name}_curves"][m], rtol=0, atol=1e-12)
        np.testing.assert_allclose(curve, g[f"{name}_curves_full"][m], rtol=0, atol=1e-10)
        sharp = O.idos_sharp_from_bands(bands, kw, lo, hi, npts, cell.area)
        np.testing.assert_allclose(sharp, g[f"{name}_sharp"][m], rtol=0, atol=1e-12)


def test_level_moments_match_reference():
    g = golden("levels.npz")
    lo, hi, npts = g["grid"]
    assert (lo, hi) == (LO_G - 0.02, HI_G + 0.02) or abs(lo - (LO_G)) < 1e-12
    cache = {}
    model = O.graphene_model()
    for level, (n, M) in enumerate(((4, 24), (8, 8)), start=1):
        res = O.sample_level(model, 16, level, n, M, 0.05, level > 1, 2026, lo, hi, int(npts), 0.01, cache=cache)
        np.testing.assert_allclose(res["full"], g[f"L{level}_full"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(res["mean"], g[f"L{level}_mean"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(res["variance"], g[f"L{level}_var"], rtol=0, atol=1e-12)


def test_energy_range_detection_graphene():
    emin, emax = O.detect_energy_range(O.graphene_model(), 32)
    assert emin - 0.02 == pytest.approx(LO_G, abs=1e-12)
    assert emax + 0.02 == pytest.approx(HI_G, abs=1e-12)


def test_fx_artifacts_present_and_consistent():
    g = golden("fx_reference_artifacts.npz")
    idos = g["rates_idos"]
    assert idos.shape == (4096, 4)
    assert idos[0, 0] == LO_G
    summary = json.loads(str(g["rates_summary_json"]))
    assert summary["config"]["levels"]["nq"] == 32
    # the unperturbed nu=16 plateau: 2 states per fundamental cell
    assert g["rates_unperturbed"][-1, 1] == pytest.approx(2.0, abs=1e-12)
