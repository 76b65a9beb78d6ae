"""GPU edge cases of every entry point: an empty batch (m = 0), the largest n on the generic
kernel (S = n_eff/2 without a ring configuration: n = 4097 odd, n = 8192), and n = 2 / 3 (a
single rotation; the bye with one real pair)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_00003_b200 as pkg
    return pkg


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("n", [2, 3, 256, 1024, 2047])
def test_empty_batch(g, n):
    """m = 0: outputs are empty, dtheta (and dphi) are exactly zero -- the gradient of a sum over
    no columns -- on the ring, unitary and GEMM paths."""
    N = n * (n - 1) // 2
    th = torch.from_numpy(synth.theta(N, seed=1)).cuda()
    X = torch.empty((n, 0), device="cuda")
    Y = g.apply(th, X)
    assert Y.shape == (n, 0)
    dth, dX = g.backward(th, Y, torch.empty((n, 0), device="cuda"))
    assert dX.shape == (n, 0) and (dth == 0).all()
    Xc = torch.empty((n, 0), dtype=torch.complex64, device="cuda")
    ph = torch.from_numpy(synth.theta(N, seed=2)).cuda()
    Yc = g.u_apply(th, ph, Xc)
    dth, dph, dXc = g.u_backward(th, ph, Yc, Xc)
    assert (dth == 0).all() and (dph == 0).all() and dXc.shape == (n, 0)
    Yg = g.gemm_apply(th, X)
    dth, dXg = g.gemm_backward(th, Yg, torch.empty((n, 0), device="cuda"))
    assert (dth == 0).all() and dXg.shape == (n, 0)


@pytest.mark.parametrize("n,m", [(4097, 3), (8192, 2)])
def test_largest_generic_sizes(g, n, m):
    """n without a ring configuration at the top of the tested range: the generic kernel (pairs
    derived per block), 8.4M / 33.5M angles."""
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=n)
    X = synth.normal_matrix(n, m, seed=n, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=n, tid=synth.TID_DY)
    tt = torch.from_numpy(th).cuda()
    Y = g.apply(tt, torch.from_numpy(X).cuda())
    X64 = X.astype(np.float64)
    assert rel(Y.cpu().numpy(), oracle.apply(n, th, X64)) <= 1e-5
    dth, dX = g.backward(tt, Y, torch.from_numpy(dY).cuda())
    dto, dXo = oracle.backward(n, th, X64, dY.astype(np.float64))
    assert rel(dth.cpu().numpy(), dto) <= 1e-4
    assert rel(dX.cpu().numpy(), dXo) <= 1e-5
