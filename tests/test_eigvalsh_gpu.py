"""Batched Hermitian eigenvalues (hx_eigvalsh_batch_device) against LAPACK (numpy.linalg.eigvalsh).

Covers the shared-memory tier (n <= 160), the two-stage banded tier (n > 160, stage-1 DMMA panels +
bulge chasing), zero-padded tails (vacancy compaction), exact degeneracies and batch mixing.
"""

import ctypes as C

import numpy as np
import pytest

from paper_1611_09784_b200 import _lib

pytestmark = pytest.mark.gpu


def rand_herm(rng, n, batch, pad=0):
    a = rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))
    a = 0.5 * (a + np.conj(np.swapaxes(a, 1, 2)))
    if pad:
        a[:, n - pad:, :] = 0
        a[:, :, n - pad:] = 0
    return a


def gpu_eigvalsh(a, b=None):
    import torch

    batch, n, _ = a.shape
    dev = torch.device("cuda", 0)

    def up(m):  # column-major complex: store M^T row-major == M column-major
        mt = np.ascontiguousarray(np.swapaxes(m, 1, 2))
        return torch.from_numpy(mt.view(np.float64).reshape(batch, n, n, 2)).to(dev)

    A = up(a)
    B = None if b is None else up(b)
    eig = torch.empty((batch, n), dtype=torch.float64, device=dev)
    st = torch.empty(batch, dtype=torch.int32, device=dev)
    ctx = _lib.Device.ctx(0)
    _lib.check(_lib.load().hx_eigvalsh_batch_device(ctx, n, batch, A.data_ptr(), 0 if B is None else B.data_ptr(),
                                                    eig.data_ptr(), st.data_ptr(),
                                                    torch.cuda.current_stream(dev).cuda_stream), "eigvalsh")
    torch.cuda.synchronize()
    return eig.cpu().numpy(), st.cpu().numpy()


@pytest.mark.parametrize("n,batch", [(5, 7), (32, 9), (100, 4), (160, 3), (161, 3), (200, 3), (257, 2), (512, 2)])
def test_random_hermitian(n, batch):
    rng = np.random.default_rng(n)
    a = rand_herm(rng, n, batch)
    got, st = gpu_eigvalsh(a)
    assert (st == 0).all()
    ref = np.linalg.eigvalsh(a)
    width = ref.max() - ref.min()
    assert np.max(np.abs(got - ref)) <= 1e-10 * width


@pytest.mark.parametrize("n,pad", [(200, 37), (300, 1), (192, 64)])
def test_zero_padded_tail(n, pad):
    rng = np.random.default_rng(7)
    a = rand_herm(rng, n, 2, pad=pad)
    got, _ = gpu_eigvalsh(a)
    ref = np.linalg.eigvalsh(a)
    assert np.max(np.abs(got - ref)) <= 1e-10 * (ref.max() - ref.min())


def test_degenerate_spectrum_banded_tier():
    rng = np.random.default_rng(3)
    n = 240
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    lam = np.repeat(np.array([-3.0, 0.0, 0.0, 1.5]), n // 4)
    a = (q * lam) @ q.conj().T
    a = 0.5 * (a + a.conj().T)
    got, _ = gpu_eigvalsh(a[None])
    assert np.max(np.abs(got[0] - np.sort(lam))) <= 1e-10 * 4.5


def test_block_diagonal_already_tridiagonal():
    n = 300
    d = np.linspace(-2, 2, n)
    e = np.full(n - 1, 0.3 + 0.4j)
    a = np.diag(d).astype(complex) + np.diag(e, -1) + np.diag(np.conj(e), 1)
    got, _ = gpu_eigvalsh(a[None])
    ref = np.linalg.eigvalsh(a)
    assert np.max(np.abs(got[0] - ref)) <= 1e-10 * (ref.max() - ref.min())


@pytest.mark.parametrize("n,batch", [(40, 3), (200, 3), (320, 2)])
def test_random_generalized(n, batch):
    """A x = lambda B x with B Hermitian positive definite (zhegv, spectrum.py:106-108): the shared / global
    kernels below n = 160, the Cholesky + banded two-stage path above."""
    import scipy.linalg as sl

    rng = np.random.default_rng(7 * n)
    a = rand_herm(rng, n, batch)
    g = rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))
    b = np.einsum("bij,bkj->bik", g, g.conj()) / n + np.eye(n)
    got, st = gpu_eigvalsh(a, b)
    assert (st == 0).all()
    for m in range(batch):
        ref = sl.eigh(a[m], b[m], eigvals_only=True)
        assert np.max(np.abs(got[m] - ref)) <= 1e-10 * (ref.max() - ref.min())
