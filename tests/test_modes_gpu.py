"""The remaining run modes natively on libhx: Engine.run_rates (runner.py:347-378)
against the reference's own rates artefact (pkg/frontend/fixtures/rates: level variances, bias proxies, fitted
W / S / D), Engine.band_structure against the oracle, and the reference CLI's "bands" mode (cli.py:132-152,
which calls spectrum.solve_bands directly) on the libhx solve installed by reference_engine.install."""

import csv
import json

import numpy as np
import pytest

import hexmc_oracle as O
from conftest import golden
from reference_pkg import import_hexmc

import paper_1611_09784_b200 as hx

pytestmark = pytest.mark.gpu


def test_native_run_rates_reproduces_reference_rates_fixture():
    g = golden("fx_reference_artifacts.npz")
    summary = json.loads(str(g["rates_summary_json"]))
    levels = json.loads(str(g["rates_levels_json"]))
    eng = hx.Engine(hx.GrapheneNNModel(), nq=32, delta=0.01, master_seed=2024, bz_mode="full", energy_points=4096)
    plan = hx.LevelPlan(ns=(4, 8, 16), samples=(24, 24, 24), nq=32, p_vac=0.0625, delta=0.01)
    res = eng.run_rates(plan, window=(-6.0, 4.0))
    np.testing.assert_allclose(res.bias_proxies, summary["bias_proxies"], rtol=1e-7, atol=0)
    for k in ("W", "S", "D"):
        assert getattr(res.rates, k.lower()).value == pytest.approx(summary["rates"][k]["value"], rel=1e-6)
    assert res.rates.mlmc_benefit == summary["mlmc_benefit"]
    for rec, ref in zip(res.records, levels):
        assert rec["set"].stats.cache_hits == ref["cache_hits"]
        assert rec["variance_q"] == pytest.approx(ref["variance_q"], rel=1e-6)
        assert rec["variance_diff"] == pytest.approx(ref["variance_diff"], rel=1e-6)


@pytest.mark.parametrize("model_kind,n,nq", [("graphene", 4, 8), ("graphene", 3, 6), ("table", 2, 4)])
def test_band_structure_vs_oracle(model_kind, n, nq):
    from conftest import TABLE

    model = hx.load_coupling_table(TABLE) if model_kind == "table" else hx.GrapheneNNModel()
    om = O.parse_table(str(TABLE)) if model_kind == "table" else O.graphene_model()
    eng = hx.Engine(model, nq=nq, delta=0.01, master_seed=1, bz_mode="full", energy_points=64)
    bands = eng.band_structure(n)
    ref = O.solve_bands(O.make_cell(om, n), om, 0, bands.grid.kpoints)
    width = ref.max() - ref.min()
    assert np.max(np.abs(bands.energies - ref)) <= 1e-10 * width


def test_reference_cli_bands_mode_on_libhx(tmp_path, monkeypatch):
    hexmc = import_hexmc()
    from paper_1611_09784_b200 import reference_engine

    monkeypatch.setattr(hexmc.cli, "solve_bands", hexmc.cli.solve_bands)  # restored after the test
    monkeypatch.setattr(hexmc.runner, "solve_bands", hexmc.runner.solve_bands)
    monkeypatch.setattr(hexmc.cli, "Engine", hexmc.cli.Engine)

    def cfg(out):
        data = {"material": {"kind": "graphene"}, "disorder": {"p_vac": 0.05, "master_seed": 3},
                "levels": {"nq": 8, "ns": [4], "samples": [1]}, "qoi": {"delta": 0.01},
                "run": {"mode": "bands", "workers": 1, "out_dir": str(out)}}
        return hexmc.config.parse_config(data)

    hexmc.cli.execute(cfg(tmp_path / "cpu"))  # the reference itself (LAPACK per k)
    cls = reference_engine.install(hexmc)

    def no_cpu_jobs(func, tasks, workers=1, task_ids=None):
        assert not list(tasks), "a job reached the reference's CPU path"
        return []

    monkeypatch.setattr(hexmc.runner, "parallel_map", no_cpu_jobs)
    monkeypatch.setattr(hexmc.spectrum, "_eigvals", lambda *a: (_ for _ in ()).throw(AssertionError("CPU solve")))
    hexmc.cli.execute(cfg(tmp_path / "gpu"))
    assert cls.gpu_batches > 0

    def rows(p):
        with open(p) as fh:
            r = list(csv.reader(fh))
        return r[0], np.array([[float(x) for x in row] for row in r[1:]])

    hg, gb = rows(tmp_path / "gpu" / "bands.csv")
    hc, cb = rows(tmp_path / "cpu" / "bands.csv")
    assert hg == hc
    np.testing.assert_array_equal(gb[:, :3], cb[:, :3])
    width = cb[:, 3].max() - cb[:, 3].min()
    assert np.max(np.abs(gb[:, 3] - cb[:, 3])) <= 1e-10 * width
    _, gu = rows(tmp_path / "gpu" / "idos.csv")
    _, cu = rows(tmp_path / "cpu" / "idos.csv")
    np.testing.assert_allclose(gu[:, 1], cu[:, 1], rtol=0, atol=1e-9)
