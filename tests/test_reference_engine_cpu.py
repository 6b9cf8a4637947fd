"""The reference-side adapter (paper_1611_09784_b200.reference_engine) keeps the reference's batch-seam
semantics: with its libhx group call replaced by the reference's own per-job evaluation, every result,
hit count and cost equals the reference Engine's evaluate_masks (runner.py:206-244) on the same requests,
and failures surface as the reference's TaskError."""

import numpy as np
import pytest

from reference_pkg import import_hexmc

from paper_1611_09784_b200.reference_engine import cuda_engine_class, to_native_model


def test_seam_semantics_match_reference_engine():
    hexmc = import_hexmc()
    R = hexmc.runner
    base = R.Engine(hexmc.GrapheneNNModel(), nq=8, delta=0.01, master_seed=3, workers=1, bz_mode="reduced",
                    energy_points=41)
    Cuda = cuda_engine_class(R.Engine)

    class Fake(Cuda):
        def _hx_group(self, n, q, masks, task_ids):  # the reference's per-job path, batched by (n, q)
            res = [R._eval_job((self.model, n, q, m, self.grid, self.delta, self.bz_mode)) for m in masks]
            return np.stack([v for v, _ in res]), np.array([0.0 for _ in res]), []

    eng = Fake(hexmc.GrapheneNNModel(), nq=8, delta=0.01, master_seed=3, workers=1, bz_mode="reduced",
               energy_points=41)
    rng = np.random.default_rng(0)
    for batch in range(3):
        reqs = [(n, 8 // n, int(rng.integers(0, 6)), (batch, i)) for i, n in enumerate([2, 4, 2, 2, 4, 4, 2])]
        a, ha, _ = base.evaluate_masks(reqs)
        b, hb, _ = eng.evaluate_masks(reqs)
        assert ha == hb
        for (va, _), (vb, _) in zip(a, b):
            np.testing.assert_array_equal(va, vb)


def test_failures_are_reference_task_errors():
    hexmc = import_hexmc()
    R = hexmc.runner
    Cuda = cuda_engine_class(R.Engine)

    class Failing(Cuda):
        def _hx_group(self, n, q, masks, task_ids):
            return np.zeros((len(masks), self.grid.npoints)), np.zeros(len(masks)), \
                [(tid, hexmc.spectrum.SolverError("eigensolver failed at k=(0, 0)")) for tid in task_ids[::-1]]

    eng = Failing(hexmc.GrapheneNNModel(), nq=4, delta=0.01, master_seed=3, workers=1, bz_mode="reduced",
                  energy_points=11)
    with pytest.raises(R.TaskError) as ei:
        eng.evaluate_masks([(2, 2, 1, "a"), (2, 2, 2, "b")])
    assert [tid for tid, _ in ei.value.failures] == ["a", "b"]  # job order, as parallel_map reports


def test_model_conversion():
    hexmc = import_hexmc()
    g = to_native_model(hexmc.GrapheneNNModel(eps_2p=0.1, t=-2.8, s=0.1))
    assert (g.eps_2p, g.t, g.s) == (0.1, -2.8, 0.1)
    with pytest.raises(TypeError):
        to_native_model(object())


def test_fit_rates_restatement_matches_reference():
    """estimators.fit_rates / fit_loglog_slope (the rates mode's host arithmetic) against the reference's own
    functions (mlmc.py:268-338) on random positive observations."""
    hexmc = import_hexmc()
    from paper_1611_09784_b200.estimators import fit_loglog_slope, fit_rates

    rng = np.random.default_rng(4)
    for nlev in (2, 3, 4):
        sizes = [4 * 2**i for i in range(nlev)]
        obs = {k: list(np.exp(rng.normal(size=nlev))) for k in ("v", "d", "w")}
        prox = list(np.exp(rng.normal(size=nlev - 1))) if nlev > 2 else None
        a = fit_rates(sizes, bias_proxies=prox, variances=obs["v"], cv_diff_variances=obs["d"], work=obs["w"])
        b = hexmc.mlmc.fit_rates(sizes, bias_proxies=prox, variances=obs["v"], cv_diff_variances=obs["d"],
                                 work=obs["w"])
        for k in ("w", "s", "d", "c"):
            x, y = getattr(a, k), getattr(b, k)
            assert (x is None) == (y is None)
            if x is not None:
                assert x.value == y.value
                assert (np.isnan(x.stderr) and np.isnan(y.stderr)) or x.stderr == y.stderr
        assert a.mlmc_benefit == b.mlmc_benefit and a.mc_benefit == b.mc_benefit
    with pytest.raises(ValueError):
        fit_loglog_slope([4, 8], [1.0, -1.0])
