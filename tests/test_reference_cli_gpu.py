"""Drop-in proof: the reference's own CLI (cli.execute, cli.py:83-265), with only its Engine's batch seam
replaced by libhx (paper_1611_09784_b200.reference_engine), reproduces the reference's committed run
artefacts (pkg/frontend/fixtures/{rates,bilevel}, parsed into tests/golden/fx_reference_artifacts.npz).
The per-job CPU path (_eval_job via parallel_map) is disabled for the run, so every curve comes from the GPU."""

import csv
import json

import numpy as np
import pytest

from conftest import golden
from reference_pkg import import_hexmc

from paper_1611_09784_b200.reference_engine import cuda_engine_class

pytestmark = pytest.mark.gpu
TOL = 1e-9


def read_csv(path):
    with open(path) as fh:
        rows = list(csv.reader(fh))
    return rows[0], np.array([[float(x) for x in r] for r in rows[1:]])


@pytest.mark.parametrize("run", ["rates", "bilevel"])
def test_reference_cli_on_gpu_engine_reproduces_fixture(run, tmp_path, monkeypatch):
    hexmc = import_hexmc()
    g = golden("fx_reference_artifacts.npz")
    ref_summary = json.loads(str(g[f"{run}_summary_json"]))
    ref_levels = json.loads(str(g[f"{run}_levels_json"]))
    data = json.loads(json.dumps(ref_summary["config"]))
    data["run"]["out_dir"] = str(tmp_path)
    data["run"]["workers"] = 1
    cfg = hexmc.config.parse_config(data)

    def no_cpu_jobs(func, tasks, workers=1, task_ids=None):
        tasks = list(tasks)
        assert not tasks, "a job reached the reference's CPU path"
        return []

    engine_cls = cuda_engine_class(hexmc.runner.Engine)
    monkeypatch.setattr(hexmc.cli, "Engine", engine_cls)
    monkeypatch.setattr(hexmc.runner, "parallel_map", no_cpu_jobs)
    summary = hexmc.cli.execute(cfg)
    assert engine_cls.gpu_batches > 0

    head, idos = read_csv(tmp_path / "idos.csv")
    assert head == ["energy_eV", "idos_mean", "idos_variance", "dos"]
    ref = g[f"{run}_idos"]
    np.testing.assert_allclose(idos[:, 0], ref[:, 0], rtol=0, atol=1e-13)
    np.testing.assert_allclose(idos[:, 1], ref[:, 1], rtol=0, atol=TOL)
    np.testing.assert_allclose(idos[:, 2], ref[:, 2], rtol=0, atol=TOL)
    np.testing.assert_allclose(idos[:, 3], ref[:, 3], rtol=0, atol=1e-6)
    _, unp = read_csv(tmp_path / "unperturbed.csv")
    np.testing.assert_allclose(unp[:, 1], g[f"{run}_unperturbed"][:, 1], rtol=0, atol=TOL)
    if f"{run}_slmc" in g.files:
        _, slmc = read_csv(tmp_path / "slmc.csv")
        np.testing.assert_allclose(slmc[:, 1], g[f"{run}_slmc"][:, 1], rtol=0, atol=TOL)
        np.testing.assert_allclose(slmc[:, 2], g[f"{run}_slmc"][:, 2], rtol=0, atol=TOL)
    levels = [json.loads(line) for line in open(tmp_path / "levels.jsonl")]
    assert len(levels) == len(ref_levels)
    for a, b in zip(levels, ref_levels):
        for k in ("level", "n", "q", "nsamples", "cache_hits"):
            assert a[k] == b[k], k
        assert a["mean_level_variance"] == pytest.approx(b["mean_level_variance"], rel=1e-6)
        for k in ("variance_q", "variance_diff"):
            if k in b:
                assert a[k] == pytest.approx(b[k], rel=1e-6)
    assert summary["levels"] == ref_summary["levels"]
    assert summary["energy_grid"]["points"] == ref_summary["energy_grid"]["points"]
    if run == "rates":
        # W (bias proxies), S (variance decay) and D (CV-difference decay) depend on the curves only;
        # C (cost) is fitted to wall time and is not compared
        for k in ("W", "S", "D"):
            if ref_summary["rates"].get(k) and summary["rates"].get(k):
                assert summary["rates"][k]["value"] == pytest.approx(ref_summary["rates"][k]["value"], rel=1e-6)
