"""Functional test of bench.py's N > 1 path on a one-GPU box: two ranks (torch.distributed.run, gloo backend,
both on cuda:0 - the collectives are host-side and the ranks' kernels never wait on each other; this checks the
plumbing, it is not a measurement).  Weak replicas: each rank draws its own replicate range, the level moments
are combined with the exact int64 all-reduce, and the device pipeline's level means must equal the public
Engine's (shard=(rank, 2)) bit for bit; split mode: the unique masks are split by sum d^3 and all-gathered."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks_on_one_gpu(scaling):
    env = dict(os.environ, HX_DIST_BACKEND="gloo", HX_BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29641" if scaling == "weak" else "--master-port=29642",
           str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1", "--no-cpu-baseline",
           "--scaling", scaling]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling
    assert d["self_check"]["bitwise_equal"], d["self_check"]
    per_step = sum(M for M in (4096, 1024, 256, 64)) * (2 if scaling == "weak" else 1)
    assert abs(d["value"] * d["ms_per_step"] * 1e-3 - per_step) <= 1e-6 * per_step
