"""World-size-2 gloo test of the N>1 host logic (CPU): per-rank replicate ranges, quarter masks and the exact
cross-rank combination of level moments (fixed-point limbs, int64 all-reduce) reproduce the single-process
level statistics BIT FOR BIT (the reference's contract: results identical for any worker count,
/root/reference/pkg/tests/test_runner.py:39-43), and agree with np.mean / np.var(ddof=1)
(mlmc.py:143-154) to rounding."""

import os
import socket
import threading
from fractions import Fraction

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_09784_b200 import _lib
from paper_1611_09784_b200.estimators import exact_level_moments
from paper_1611_09784_b200.geometry import build_supercell, partition_quarters
from paper_1611_09784_b200.models import GrapheneNNModel
from paper_1611_09784_b200.sampling import restrict_words, sample_masks

M, NU, P, SEED, LEVEL = 40, 8, 0.05, 2026, 2


def fake_curve(words):
    # deterministic stand-in for a per-sample IDOS curve (the GPU path is tested in -m gpu)
    x = np.linspace(0, 1, 17)
    h = np.array([bin(int(w)).count("1") for w in words.reshape(-1)]).sum()
    return np.sin(x * (1 + h)) * 1e-3 + 0.37 * h


def rank_curves(rank, m=M):
    sc = build_supercell(GrapheneNNModel().lattice_spec(), NU)
    words = sample_masks(sc.nunits, P, SEED, LEVEL, rank * m, m)  # replicate range of this rank
    sub = restrict_words(words, partition_quarters(sc))
    full = np.stack([fake_curve(words[i]) for i in range(m)])
    quarters = np.stack([[fake_curve(sub[i, r]) for r in range(4)] for i in range(m)])
    return full, quarters


def worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full, quarters = rank_curves(rank)
    mean, var = exact_level_moments(full, quarters, world * M, allreduce=dist.all_reduce)
    out.put((rank, mean, var))
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_exact_moments_bitwise_equal_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (m, v)) for r, m, v in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single process over the union of both replicate ranges (= replicates [0, 2M) of the stream)
    full, quarters = rank_curves(0, 2 * M)
    mean1, var1 = exact_level_moments(full, quarters, 2 * M)
    for r in range(2):
        assert np.array_equal(got[r][0], mean1) and np.array_equal(got[r][1], var1)
    terms = full - 0.25 * (((quarters[:, 0] + quarters[:, 1]) + quarters[:, 2]) + quarters[:, 3])
    np.testing.assert_allclose(mean1, terms.mean(0), rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(var1, terms.var(0, ddof=1), rtol=1e-12, atol=0)


def test_fixed_sums_independent_of_split_and_order():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((257, 9)) * np.exp(rng.uniform(-30, 12, (257, 9)))
    total = _lib.fixed_sums(x)
    perm = rng.permutation(257)
    parts = [_lib.fixed_sums(x[perm[a:b]]) for a, b in ((0, 13), (13, 100), (100, 257))]
    assert np.array_equal(parts[0] + parts[1] + parts[2], total)
    v = _lib.fixed_finalize(total, 1.0)
    ref = np.array([float(sum(map(Fraction, x[:, j]))) for j in range(9)])
    np.testing.assert_allclose(v, ref, rtol=1e-15, atol=2.0**-100)


def test_single_sample_variance_is_nan():
    mean, var = exact_level_moments(np.ones((1, 5)) * 0.5, None, 1)
    assert np.all(mean == 0.5) and np.all(np.isnan(var))


def test_replica_ranges_are_disjoint_streams():
    sc = build_supercell(GrapheneNNModel().lattice_spec(), 4)
    a = sample_masks(sc.nunits, 0.3, SEED, 1, 0, 8)
    b = sample_masks(sc.nunits, 0.3, SEED, 1, 8, 8)
    both = sample_masks(sc.nunits, 0.3, SEED, 1, 0, 16)
    np.testing.assert_array_equal(np.concatenate([a, b]), both)


def split_worker(rank, world, port, out):
    """Engine(shard_mode="split") host logic with gloo: d^3-balanced slices, ordered all-gathers from concurrent
    pieces, stitching in row order.  The solve itself is replaced by a deterministic per-row function (the GPU
    solve is covered by the -m gpu tests)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from concurrent.futures import ThreadPoolExecutor

    from paper_1611_09784_b200.engine import Engine

    eng = Engine.__new__(Engine)
    eng.shard, eng.shard_mode, eng.device, eng.io_bytes = (rank, world), "split", 0, [0, 0]
    eng.grid = type("G", (), {"npoints": 7})()
    eng._coll = threading.Condition()
    eng._coll_turn = 0
    sc = build_supercell(GrapheneNNModel().lattice_spec(), NU)
    eng.cell = lambda n, device=None: type("C", (), {"kept_dims": staticmethod(
        lambda w: 2 * NU * NU - np.array([sum(bin(int(x)).count("1") for x in r) for r in w]))})()
    seen = []

    def fake_solve(n, q, words, ids, ctx=None, device=None):
        seen.append(len(words))
        return np.stack([np.full(7, words_to_float(r)) for r in words]), 0.5

    eng._solve_group = fake_solve
    groups = [sample_masks(sc.nunits, P, SEED, lvl, 0, cnt) for lvl, cnt in ((1, 40), (2, 3), (3, 1), (4, 17))]
    with ThreadPoolExecutor(max_workers=len(groups)) as ex:
        futs = [ex.submit(eng._solve_split, NU, 1, g, list(range(len(g))), None, False, t)
                for t, g in enumerate(groups)]
        res = [f.result() for f in futs]
    out.put((rank, [r[0] for r in res], seen))
    dist.destroy_process_group()


def words_to_float(row):
    return float(sum(int(w) % 1000003 for w in row))


def test_two_rank_split_mode_stitches_every_group():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=split_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (c, s)) for r, c, s in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = build_supercell(GrapheneNNModel().lattice_spec(), NU)
    for gi, (lvl, cnt) in enumerate(((1, 40), (2, 3), (3, 1), (4, 17))):
        words = sample_masks(sc.nunits, P, SEED, lvl, 0, cnt)
        want = np.stack([np.full(7, words_to_float(r)) for r in words])
        for r in range(2):
            np.testing.assert_array_equal(got[r][0][gi], want)
    # both ranks solved a share of the 40-row group
    assert sum(got[0][1]) + sum(got[1][1]) == 40 + 3 + 1 + 17
