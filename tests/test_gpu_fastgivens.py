"""GPU parity of the fast (square-root-free) Givens variant against
the fp64 oracle: the same Y = U(theta) X and U as the three-shear path, on every one-lane ring
configuration (n_eff = 8, 16, 32, 64, odd n with the bye), with masks, wide-range angles, ragged
and large batches; other n are refused (GIVENS_EUNSUPPORTED)."""
import numpy as np
import pytest
import torch

import oracle
from _parity import rel
import synth

pytestmark = pytest.mark.gpu

TOL_Y = 1e-5


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_00003_b200 as pkg
    return pkg


def _cuda(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


FG_N = [7, 8, 15, 16, 31, 32, 63, 64]


@pytest.mark.parametrize("n", FG_N)
@pytest.mark.parametrize("m", [1, 37, 300, 5000])
def test_fast_apply_parity(g, n, m):
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=n + m)
    X = synth.normal_matrix(n, m, seed=n, tid=synth.TID_X)
    Y = g.fast_apply(_cuda(th), _cuda(X)).cpu().numpy()
    assert rel(Y, oracle.apply(n, th, X.astype(np.float64))) <= TOL_Y


@pytest.mark.parametrize("n", FG_N)
def test_fast_build_U_parity(g, n):
    th = synth.theta(n * (n - 1) // 2, seed=3 * n, half_range=8 * np.pi)
    U = g.fast_build_U(_cuda(th), n).cpu().numpy()
    assert np.abs(U - oracle.build_U(n, th)).max() <= 1e-5 * np.sqrt(n)


@pytest.mark.parametrize("n", [8, 31, 64])
def test_fast_masked_wide_angles(g, n):
    N = n * (n - 1) // 2
    m = 129
    th = synth.theta(N, seed=n, half_range=8 * np.pi)
    th[::7] = np.float32(np.pi / 2)  # |cos| ~ 0: the second factoring
    th[1::11] = np.float32(np.pi)
    mask = synth.random_mask(N, 0.6, seed=n)
    th_nan = th.copy()
    th_nan[mask == 0] = np.nan
    X = synth.normal_matrix(n, m, seed=n, tid=synth.TID_X)
    Y = g.fast_apply(_cuda(th_nan), _cuda(X), mask=_cuda(mask)).cpu().numpy()
    assert rel(Y, oracle.apply(n, th, X.astype(np.float64), mask=mask)) <= TOL_Y


def test_fast_matches_three_shear(g):
    """Both factorisations of the same product: Y agrees to fp32 rounding on a large batch."""
    n, m = 64, 65536
    th = _cuda(synth.theta(n * (n - 1) // 2, seed=1))
    X = _cuda(synth.normal_matrix(n, m, seed=1, tid=synth.TID_X))
    Yf, Ys = g.fast_apply(th, X), g.apply(th, X)
    assert rel(Yf.cpu().numpy(), Ys.cpu().numpy()) <= 2e-6


@pytest.mark.parametrize("n", [2, 6, 65, 256])
def test_fast_unsupported(g, n):
    th = torch.zeros(n * (n - 1) // 2, device="cuda")
    with pytest.raises(g.GivensError):
        g.fast_apply(th, torch.zeros(n, 4, device="cuda"))
