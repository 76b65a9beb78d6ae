"""GPU parity for the GEMM path: U-build on the register ring + 3xTF32 tensor-core
GEMMs + Algorithm 3 on Gamma, through the C ABI (givens_gemm_apply / givens_gemm_backward), against
the fp64 oracle. Same tolerances as the ring path (BASELINE.json north_star). Includes the full C3
configuration (n=1024, m=65536) against a full oracle backward, for both paths."""
import numpy as np
import pytest
import torch

import oracle
from _parity import rel
import synth

pytestmark = pytest.mark.gpu

TOL_Y = 1e-5
TOL_DTH = 1e-4


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_00003_b200 as pkg
    return pkg




def _cuda(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n", [2, 3, 8, 33, 100, 256, 1024, 1120, 2047])
@pytest.mark.parametrize("m", [1, 45, 300])
def test_gemm_path_parity(g, n, m):
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=n + m)
    X = synth.normal_matrix(n, m, seed=n, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=n, tid=synth.TID_DY)
    tt, Xt, dYt = _cuda(th), _cuda(X), _cuda(dY)
    ws = g.gemm_workspace(n, m)
    Y = g.gemm_apply(tt, Xt, ws=ws)
    X64 = X.astype(np.float64)
    assert rel(Y.cpu().numpy(), oracle.apply(n, th, X64)) <= TOL_Y
    dth, dX = g.gemm_backward(tt, Y, dYt, ws=ws, recompute=False)
    dto, dXo = oracle.backward(n, th, X64, dY.astype(np.float64))
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y
    Yt = g.gemm_apply(tt, Xt, transpose=True)
    assert rel(Yt.cpu().numpy(), oracle.apply(n, th, X64, transpose=True)) <= TOL_Y


@pytest.mark.parametrize("n", [9, 256, 2047])
def test_gemm_path_mask_and_layout(g, n):
    rng = np.random.default_rng(n)
    p = rng.permutation(n + n % 2).astype(np.int32)
    lay = g.Layout(n, perm=p, reflect_col=n // 2)
    mask = g.mask_from_keep(n, n // 2, perm=p)
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=3)
    X = synth.normal_matrix(n, 50, seed=3, tid=synth.TID_X)
    dY = synth.normal_matrix(n, 50, seed=3, tid=synth.TID_DY)
    Y = g.gemm_apply(_cuda(th), _cuda(X), mask=_cuda(mask), layout=lay)
    X64 = X.astype(np.float64)
    assert rel(Y.cpu().numpy(), oracle.apply(n, th, X64, mask, perm=p, reflect=n // 2)) <= TOL_Y
    dth, dX = g.gemm_backward(_cuda(th), Y, _cuda(dY), mask=_cuda(mask), layout=lay)
    dto, dXo = oracle.backward(n, th, X64, dY.astype(np.float64), mask, perm=p, reflect=n // 2)
    dth = dth.cpu().numpy()
    assert (dth[mask == 0] == 0).all()
    assert rel(dth, dto) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


@pytest.fixture(scope="module")
def c3():
    """C3 inputs and the fp64 oracle's full forward on sampled columns and full backward (the
    dtheta sum over all 65536 columns; ~20 s on the host cores)."""
    n, m = 1024, 65536
    th = synth.theta(n * (n - 1) // 2, seed=21)
    X = synth.normal_matrix(n, m, seed=21, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=21, tid=synth.TID_DY)
    dto, _ = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64), want_dX=False)
    cols = np.unique(np.concatenate([np.arange(4), np.random.default_rng(1).integers(0, m, 12), [m - 1]]))
    Yo = oracle.apply(n, th, X[:, cols].astype(np.float64))
    _, dXo = oracle.backward(n, th, X[:, cols].astype(np.float64), dY[:, cols].astype(np.float64))
    return n, m, th, X, dY, dto, cols, Yo, dXo


@pytest.mark.parametrize("path", ["ring", "gemm"])
def test_c3_full_dtheta_vs_oracle(g, c3, path):
    """C3 at full size in the bench configuration: every dtheta (a sum over all 65536 columns) vs
    the oracle's, Y and dX on sampled columns."""
    n, m, th, X, dY, dto, cols, Yo, dXo = c3
    tt, Xt, dYt = _cuda(th), _cuda(X), _cuda(dY)
    if path == "ring":
        Y = g.apply(tt, Xt)
        dth, dX = g.backward(tt, Y, dYt)
    else:
        ws = g.gemm_workspace(n, m)
        Y = g.gemm_apply(tt, Xt, ws=ws)
        dth, dX = g.gemm_backward(tt, Y, dYt, ws=ws, recompute=False)
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(Y.cpu().numpy()[:, cols], Yo) <= TOL_Y
    assert rel(dX.cpu().numpy()[:, cols], dXo) <= TOL_Y


def test_gemm_path_errors(g):
    n, m = 16, 8
    th = torch.zeros(n * (n - 1) // 2, device="cuda")
    X = torch.zeros(n, m, device="cuda")
    with pytest.raises(g.GivensError):
        g.gemm_apply(th, X, out=X)  # no aliasing on the GEMM path
    with pytest.raises(g.GivensError):
        g.gemm_apply(th, X, ws=torch.empty(256, dtype=torch.uint8, device="cuda"))
