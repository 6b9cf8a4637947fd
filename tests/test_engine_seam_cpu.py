"""Host logic of the batch seam (Engine._evaluate_batches) without a GPU: the solver is replaced by a
deterministic fake, and the dedup / placement / hit / cost accounting is checked against a literal
restatement of the reference's evaluate_masks loop (runner.py:206-244), called batch after batch."""

import numpy as np
import pytest

import paper_1611_09784_b200 as hx
from paper_1611_09784_b200 import _lib
from paper_1611_09784_b200 import engine as E

LO, HI = -6.580201874549387, 14.863393148450246


def fake_curve(n, q, row, npts):
    h = np.frombuffer(np.asarray(row, dtype=np.uint64).tobytes(), dtype=np.uint8).astype(np.float64)
    return np.full(npts, float(n * 1000 + q)) + np.arange(npts) * 1e-3 + h.sum()


class FakeEngine(hx.Engine):
    def _solve_group(self, n, q, words, task_ids, ctx=None):
        assert len(task_ids) == len(words)
        return np.stack([fake_curve(n, q, w, self.grid.npoints) for w in words]), 0.5


@pytest.fixture
def engine(monkeypatch):
    monkeypatch.setattr(_lib.Device, "lane", classmethod(lambda cls, d, i, high=None: None))
    return FakeEngine(hx.GrapheneNNModel(), nq=16, delta=0.01, master_seed=7, bz_mode="reduced", rng="host",
                      energy_points=11, energy_range=(LO + 0.02, HI - 0.02))


def reference_accounting(batches, npts):
    """The reference loop: key (n, q, mask) against the run cache, then against earlier requests of the
    same batch; new jobs cost 0.5 each (the fake per-job time)."""
    cache = {}
    out = []
    for groups in batches:
        hits, spent, pending = 0, 0.0, {}
        res = []
        for n, q, words in groups:
            cu = []
            for row in words:
                k = (n, q, row.tobytes())
                if k in cache or k in pending:
                    hits += 1
                else:
                    pending[k] = fake_curve(n, q, row, npts)
                    spent += 0.5
                cu.append(cache[k] if k in cache else pending[k])
            res.append(np.stack(cu))
        cache.update(pending)
        out.append((res, hits, spent))
    return out


def test_batches_match_sequential_reference(engine):
    rng = np.random.default_rng(3)
    # small alphabets so that in-batch and cross-batch duplicates are common
    b1 = [(4, 4, rng.integers(0, 4, size=(40, 1)).astype(np.uint64)),
          (2, 8, rng.integers(0, 3, size=(30, 1)).astype(np.uint64))]
    b2 = [(4, 4, rng.integers(0, 6, size=(25, 1)).astype(np.uint64)),
          (8, 2, rng.integers(0, 5, size=(20, 1)).astype(np.uint64))]
    b3 = [(2, 8, rng.integers(0, 5, size=(35, 1)).astype(np.uint64))]
    batches = [b1, b2, b3]
    ids = lambda gi, new, inv: [("t", int(i)) for i in new]  # noqa: E731
    got = engine._evaluate_batches([(b, ids) for b in batches])
    want = reference_accounting(batches, engine.grid.npoints)
    for (gres, ghits, gspent), (wres, whits, wspent) in zip(got, want):
        assert ghits == whits
        assert gspent == pytest.approx(wspent)
        for (cu, pj), wc in zip(gres, wres):
            np.testing.assert_array_equal(cu, wc)
    # a second call hits the run cache for everything
    again = engine._evaluate_batches([(b1, ids)])[0]
    assert again[1] == 70 and again[2] == 0.0


def test_run_mlmc_equals_levels_in_order(engine, monkeypatch):
    monkeypatch.setattr(E, "level_moments", lambda full, quarters, device, want_terms=True: _np_moments(full, quarters))
    plan = hx.LevelPlan(ns=(2, 4, 8), samples=(64, 32, 8), nq=16, p_vac=0.2, delta=0.01)
    _, sets = engine.run_mlmc(plan)
    seq = FakeEngine(hx.GrapheneNNModel(), nq=16, delta=0.01, master_seed=7, bz_mode="reduced", rng="host",
                     energy_points=11, energy_range=(LO + 0.02, HI - 0.02))
    for lvl, (n, m) in enumerate(zip(plan.ns, plan.samples), start=1):
        s = seq.sample_level(lvl, n, m, plan.p_vac, lvl > 1)
        t = sets[lvl - 1]
        assert s.stats.cache_hits == t.stats.cache_hits
        assert s.stats.wall_seconds == pytest.approx(t.stats.wall_seconds)
        np.testing.assert_array_equal(s.full, t.full)


def _np_moments(full, quarters):
    import torch

    terms = full if quarters is None else full - quarters.sum(axis=1) * 0.25
    t = torch.from_numpy(np.ascontiguousarray(terms))
    return t, t.mean(0), t.var(0) if len(terms) > 1 else t.mean(0)


def test_unique_rows_matches_numpy_axis0_unique():
    """The seam's row dedup (engine.unique_rows / first_rows) equals np.unique(axis=0) - same lexicographic
    order of the unique masks, same inverse - and the first-occurrence map of the reference loop."""
    from paper_1611_09784_b200.engine import first_rows, unique_rows

    rng = np.random.default_rng(7)
    for w in (1, 2, 4):
        for R in (1, 3, 257, 2048):
            words = (rng.integers(0, 5, size=(R, w)).astype(np.uint64) << np.uint64(61)) | np.uint64(3)
            u0, i0 = np.unique(words, axis=0, return_inverse=True)
            u1, i1 = unique_rows(words)
            assert np.array_equal(u0, u1) and np.array_equal(i0.reshape(-1), i1)
            first = np.full(i1.max() + 1, -1)
            for r in range(R - 1, -1, -1):
                first[i1[r]] = r
            assert np.array_equal(first, first_rows(i1))
    u, i = unique_rows(np.zeros((0, 2), dtype=np.uint64))
    assert u.shape == (0, 2) and i.shape == (0,)
