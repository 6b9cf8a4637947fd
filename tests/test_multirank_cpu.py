"""World-size-2 gloo test of the N>1 host logic (CPU): per-rank replicate ranges, quarter masks and the
cross-rank combination of level sums reproduce the single-process level statistics."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_09784_b200.estimators import moments_from_sums
from paper_1611_09784_b200.geometry import build_supercell, partition_quarters
from paper_1611_09784_b200.models import GrapheneNNModel
from paper_1611_09784_b200.sampling import restrict_words, sample_masks

M, NU, P, SEED, LEVEL = 40, 8, 0.05, 2026, 2


def fake_curve(words):
    # deterministic stand-in for a per-sample IDOS curve (the GPU path is tested in -m gpu)
    x = np.linspace(0, 1, 17)
    h = np.array([bin(int(w)).count("1") for w in words.reshape(-1)]).sum()
    return np.sin(x * (1 + h)) + h


def rank_sums(rank, world):
    sc = build_supercell(GrapheneNNModel().lattice_spec(), NU)
    words = sample_masks(sc.nunits, P, SEED, LEVEL, rank * M, M)  # weak-scaling replica range
    sub = restrict_words(words, partition_quarters(sc))
    terms = np.stack([fake_curve(words[m]) - 0.25 * sum(fake_curve(sub[m, r]) for r in range(4)) for m in range(M)])
    return terms.sum(0), (terms * terms).sum(0), terms


def worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s1, s2, _ = rank_sums(rank, world)
    t = torch.from_numpy(np.concatenate([s1, s2]))
    dist.all_reduce(t)
    if rank == 0:
        out.put(t.numpy())
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_level_sums_match_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    red = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    npts = red.size // 2
    mean, var = moments_from_sums(red[:npts], red[npts:], 2 * M)
    # single process over the union of both replicate ranges
    t0 = rank_sums(0, 2)[2]
    t1 = rank_sums(1, 2)[2]
    allt = np.concatenate([t0, t1])
    np.testing.assert_allclose(mean, allt.mean(0), rtol=0, atol=1e-12)
    np.testing.assert_allclose(var, allt.var(0, ddof=1), rtol=1e-9, atol=1e-12)


def test_replica_ranges_are_disjoint_streams():
    sc = build_supercell(GrapheneNNModel().lattice_spec(), 4)
    a = sample_masks(sc.nunits, 0.3, SEED, 1, 0, 8)
    b = sample_masks(sc.nunits, 0.3, SEED, 1, 8, 8)
    both = sample_masks(sc.nunits, 0.3, SEED, 1, 0, 16)
    np.testing.assert_array_equal(np.concatenate([a, b]), both)
