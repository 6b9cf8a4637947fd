"""CPU-side checks of the C-ABI boundary and the host logic (no GPU compute)."""

import re

import numpy as np
import pytest

import hexmc_oracle as O
from conftest import ROOT, TABLE, golden, words_to_int

from paper_1611_09784_b200 import _lib
from paper_1611_09784_b200.geometry import build_supercell, partition_quarters
from paper_1611_09784_b200.models import GrapheneNNModel, _csr, compile_cell, load_coupling_table
from paper_1611_09784_b200.sampling import keys_from_words, restrict_words, sample_masks, words_from_keys


def header_symbols():
    text = (ROOT / "include" / "hx.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(hx_\w+)\s*\(", text, flags=re.M)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(_lib.EXPORTED)
    header_version = int(re.search(r"#define HX_ABI_VERSION (\d+)", (ROOT / "include" / "hx.h").read_text()).group(1))
    assert lib.hx_abi_version() == header_version


def test_no_device_is_reported_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.HxError):
        _lib.Device.ctx(0)


def test_host_uniforms_bit_exact_with_reference_draws():
    g = golden("rng.npz")
    for idx in range(0, len(g["streams"]), 3):
        s, lv, r = (int(x) for x in g["streams"][idx])
        if s >= 2**64:
            continue
        np.testing.assert_array_equal(_lib.uniforms(s, lv, r, 16), g["draws"][idx])


@pytest.mark.parametrize("nu", [1, 2, 4, 8, 16, 32])
def test_host_masks_bit_identical_with_reference(nu):
    words = golden("rng.npz")[f"graphene_nu{nu}"]
    got = sample_masks(2 * nu * nu, 0.05, 2026, 1 + (nu % 5), 0, len(words))
    np.testing.assert_array_equal(got, words)


def test_masks_random_streams_match_numpy():
    rng = np.random.default_rng(5)
    for _ in range(20):
        seed = int(rng.integers(0, 2**63))
        level = int(rng.integers(0, 2**31))
        rep = int(rng.integers(0, 2**31))
        nunits = int(rng.integers(1, 300))
        p = float(rng.uniform(0, 1))
        got = sample_masks(nunits, p, seed, level, rep, 1)
        assert words_to_int(got[0]) == O.sample_mask(nunits, p, seed, level, rep)


def test_key_word_roundtrip():
    keys = [0, 1, (1 << 127) | 5, (1 << 200) - 1]
    assert keys_from_words(words_from_keys(keys, 201)) == keys


@pytest.mark.parametrize("nu", [2, 4, 8])
def test_quarter_restriction_matches_oracle(nu):
    spec = GrapheneNNModel().lattice_spec()
    sc = build_supercell(spec, nu)
    part = partition_quarters(sc)
    words = sample_masks(sc.nunits, 0.3, 77, 2, 0, 16)
    sub = restrict_words(words, part)
    ocell = O.Cell(nu)
    assign, umap = O.quarter_maps(ocell)
    for m in range(16):
        key = words_to_int(words[m])
        for r in range(1, 5):
            assert words_to_int(sub[m, r - 1]) == O.restrict_mask(key, assign, umap, r)


@pytest.mark.parametrize("table,nu", [(False, 1), (False, 3), (False, 4), (True, 1), (True, 2)])
def test_instance_tables_match_oracle(table, nu):
    model = load_coupling_table(TABLE) if table else GrapheneNNModel()
    omodel = O.parse_table(TABLE) if table else O.graphene_model()
    sc = build_supercell(model.lattice_spec(), nu)
    cell = compile_cell(model, sc)
    ocell = O.make_cell(omodel, nu)
    src, dst, amp, disp = O.expand(ocell, omodel["hops"])
    np.testing.assert_array_equal(cell.h[0], src)
    np.testing.assert_array_equal(cell.h[1], dst)
    np.testing.assert_array_equal(cell.h[2], amp)
    np.testing.assert_allclose(cell.h[3], disp, rtol=0, atol=1e-15)
    np.testing.assert_array_equal(cell.onsite, O.onsite_vector(ocell, omodel))
    ptr, col, a, d = _csr(cell.dim, *cell.h)
    assert ptr[-1] == len(src)
    # CSR rows keep the reference's instance order per source dof
    for r in range(cell.dim):
        np.testing.assert_array_equal(col[ptr[r]:ptr[r + 1]], dst[src == r])


def test_pencil_kinds():
    g = compile_cell(GrapheneNNModel(), build_supercell(GrapheneNNModel().lattice_spec(), 2))
    assert g.pencil == _lib.HX_PENCIL_COMMUTING
    t = load_coupling_table(TABLE)
    tc = compile_cell(t, build_supercell(t.lattice_spec(), 2))
    assert tc.pencil == _lib.HX_PENCIL_STANDARD
    assert tc.dim == 44 and tc.supercell.nunits == 4


@pytest.mark.parametrize("n,q", [(4, 8), (8, 4), (16, 2), (32, 1), (4, 6), (3, 5)])
def test_time_reversal_pairs_of_the_reference_grid(n, q):
    """k -> -k classes of the reduced q x q grid (spectrum.py:59-84): multiplicities sum to q^2, the
    invariant points are the 4 (q even) or 1 (q odd) TRIMs, and every merged point's partner is its negative
    modulo the supercell reciprocal lattice."""
    from paper_1611_09784_b200.models import GrapheneNNModel
    from paper_1611_09784_b200.solver import make_bz_grid, time_reversal_reduce

    spec = GrapheneNNModel().lattice_spec()
    kp = make_bz_grid(spec, n, q, "reduced").kpoints
    reps, mult = time_reversal_reduce(spec, n, kp)
    assert mult.sum() == q * q
    assert (mult == 1).sum() == (min(q, 2) ** 2 if q % 2 == 0 else 1)
    b1, b2 = spec.reciprocal_vectors()
    B = np.stack([np.asarray(b1) / n, np.asarray(b2) / n], axis=1)
    frac = np.linalg.solve(B, kp.T).T
    for r in np.linalg.solve(B, reps.T).T:
        partners = [f for f in frac if np.allclose(np.mod(f + r + 1e-12, 1.0), 0.0, atol=1e-9)
                    or np.allclose(np.mod(f + r + 1e-12, 1.0), 1.0, atol=1e-9)]
        assert len(partners) == 1


@pytest.mark.parametrize("n,n2", [(2, 3), (4, 8), (3, 1)])
def test_rectangular_supercell_tables_match_oracle(n, n2):
    """n x n2 supercells (config-5 sizes 64 / 256 / 1024): site order, instance tables, area."""
    model = GrapheneNNModel()
    sc = build_supercell(model.lattice_spec(), n, n2)
    cell = compile_cell(model, sc)
    ocell = O.make_cell(O.graphene_model(), n, n2)
    assert cell.dim == ocell.dim == 2 * n * n2 and sc.area == pytest.approx(ocell.area, rel=1e-14)
    src, dst, amp, disp = O.expand(ocell, O.graphene_model()["hops"])
    np.testing.assert_array_equal(cell.h[0], src)
    np.testing.assert_array_equal(cell.h[1], dst)
    np.testing.assert_allclose(cell.h[3], disp, rtol=0, atol=1e-15)
    assert build_supercell(model.lattice_spec(), n, n).n2 is None  # square stays the reference's cell
