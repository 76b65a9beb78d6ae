"""GPU parity for angles outside (-pi, pi]: the paper's angles are unrestricted reals
(theta in R^N; the entries of G^e are cos/sin of theta). The
kernels reduce every angle modulo 2 pi (fp64 remainder) before the pi-flip of DESIGN.md §3, so the
shear coefficient tan(phi/2) stays bounded; without that, theta = 2 pi gave a wrong rotation.

Covers every kernel family (register ring, idle-lane ring, multi-warp ring, generic), the unitary
variant (theta and phi wide), the layout options, and the GEMM path (through build_U), at C1, C2 and
C4-like n and a C3 column sample, with theta ~ U(-8 pi, 8 pi) and with the special values
{+-pi/2, +-pi, +-3pi/2, +-2pi, +-4pi, 1e3, -1e4} spread over the angles."""
import numpy as np
import pytest
import torch

import oracle
from _parity import rel
import synth

pytestmark = pytest.mark.gpu

TOL_Y = 1e-5
TOL_DTH = 1e-4

SPECIAL = np.array([np.pi / 2, -np.pi / 2, np.pi, -np.pi, 1.5 * np.pi, -1.5 * np.pi, 2 * np.pi, -2 * np.pi,
                    4 * np.pi, -4 * np.pi, 1e3, -1e4, 6.25, 6.0, -6.2831], dtype=np.float32)


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_00003_b200 as pkg
    return pkg


def _cuda(a):
    if a is None:
        return None
    if np.iscomplexobj(a):
        a = a.astype(np.complex64)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _theta(N, kind, seed):
    if kind == "wide":
        return synth.theta(N, seed=seed, half_range=8 * np.pi)
    th = synth.theta(N, seed=seed, half_range=8 * np.pi)
    idx = np.random.default_rng(seed).permutation(N)
    k = min(N, 4 * SPECIAL.size)
    th[idx[:k]] = np.resize(SPECIAL, k)  # every special value at several (block, slot) positions
    return th


# ring (8, 256, 1024), idle-lane (48, 1120), multi-warp (2047, 4096), generic (5, 100), odd (7, 33)
AN = [2, 3, 5, 7, 8, 33, 48, 100, 256, 1024, 1120, 2047, 4096]


@pytest.mark.parametrize("kind", ["wide", "special"])
@pytest.mark.parametrize("n", AN)
def test_wide_angle_apply_backward(g, n, kind):
    m = 37 if n < 2047 else 9
    N = n * (n - 1) // 2
    th = _theta(N, kind, seed=n)
    X = synth.normal_matrix(n, m, seed=n, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=n, tid=synth.TID_DY)
    tt, Xt = _cuda(th), _cuda(X)
    X64 = X.astype(np.float64)
    Y = g.apply(tt, Xt)
    assert rel(Y.cpu().numpy(), oracle.apply(n, th, X64)) <= TOL_Y
    Yt = g.apply(tt, Xt, transpose=True)
    assert rel(Yt.cpu().numpy(), oracle.apply(n, th, X64, transpose=True)) <= TOL_Y
    dth, dX = g.backward(tt, Y, _cuda(dY))
    dto, dXo = oracle.backward(n, th, X64, dY.astype(np.float64))
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


@pytest.mark.parametrize("n", [8, 64, 256, 1024])
def test_wide_angle_build_U(g, n):
    th = _theta(n * (n - 1) // 2, "special", seed=3 * n)
    U = g.build_U(_cuda(th), n).cpu().numpy()
    assert np.abs(U - oracle.build_U(n, th)).max() <= 1e-5 * np.sqrt(n)


def test_multiples_of_two_pi_are_identity(g):
    """theta = 2 pi k (as fp32) is a rotation by the fp32 rounding residue only: U ~ I."""
    n = 64
    N = n * (n - 1) // 2
    k = np.arange(N) % 9 - 4
    th = (2 * np.pi * k).astype(np.float32)
    U = g.build_U(_cuda(th), n).cpu().numpy()
    assert np.abs(U - oracle.build_U(n, th)).max() <= 1e-5 * np.sqrt(n)
    assert np.abs(U - np.eye(n)).max() <= 1e-4


def test_wide_angle_masked(g):
    n, m = 256, 50
    N = n * (n - 1) // 2
    th = _theta(N, "special", seed=7)
    mask = synth.random_mask(N, 0.6, seed=7)
    X = synth.normal_matrix(n, m, seed=7, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=7, tid=synth.TID_DY)
    tt, mt = _cuda(th), _cuda(mask)
    Y = g.apply(tt, _cuda(X), mask=mt)
    dth, dX = g.backward(tt, Y, _cuda(dY), mask=mt)
    X64 = X.astype(np.float64)
    assert rel(Y.cpu().numpy(), oracle.apply(n, th, X64, mask=mask)) <= TOL_Y
    dto, dXo = oracle.backward(n, th, X64, dY.astype(np.float64), mask=mask)
    d = dth.cpu().numpy()
    assert (d[mask == 0] == 0).all()
    assert rel(d, dto) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


@pytest.mark.parametrize("n", [7, 33, 256, 1024, 2047])
def test_wide_angle_layout(g, n):
    p = np.random.default_rng(n).permutation(n + n % 2).astype(np.int32)
    c = n // 3
    lay = g.Layout(n, perm=p, reflect_col=c)
    m = 21
    th = _theta(n * (n - 1) // 2, "special", seed=n + 5)
    X = synth.normal_matrix(n, m, seed=n, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=n, tid=synth.TID_DY)
    tt = _cuda(th)
    X64 = X.astype(np.float64)
    Y = g.apply(tt, _cuda(X), layout=lay)
    assert rel(Y.cpu().numpy(), oracle.apply(n, th, X64, perm=p, reflect=c)) <= TOL_Y
    dth, dX = g.backward(tt, Y, _cuda(dY), layout=lay)
    dto, dXo = oracle.backward(n, th, X64, dY.astype(np.float64), perm=p, reflect=c)
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


def _c(n, m, seed, tid):
    return (synth.normal_matrix(n, m, seed, tid).astype(np.float64)
            + 1j * synth.normal_matrix(n, m, seed + 7919, tid).astype(np.float64))


@pytest.mark.parametrize("n", [5, 8, 48, 256, 1024, 2047])
def test_wide_angle_unitary(g, n):
    m = 19
    N = n * (n - 1) // 2
    th = _theta(N, "special", seed=n)
    ph = _theta(N, "wide", seed=n + 1)
    X = _c(n, m, n, synth.TID_X)
    G = _c(n, m, n, synth.TID_DY)
    Y = g.u_apply(_cuda(th), _cuda(ph), _cuda(X))
    assert rel(Y.cpu().numpy(), oracle.u_apply(n, th, ph, X)) <= TOL_Y
    dth, dph, dX = g.u_backward(_cuda(th), _cuda(ph), Y, _cuda(G))
    dto, dpo, dXo = oracle.u_backward(n, th, ph, X, G)
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dph.cpu().numpy(), dpo) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


@pytest.mark.parametrize("n", [33, 256, 1024])
def test_wide_angle_gemm_path(g, n):
    m = 45
    th = _theta(n * (n - 1) // 2, "special", seed=n + 2)
    X = synth.normal_matrix(n, m, seed=n, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=n, tid=synth.TID_DY)
    X64 = X.astype(np.float64)
    Y = g.gemm_apply(_cuda(th), _cuda(X))
    assert rel(Y.cpu().numpy(), oracle.apply(n, th, X64)) <= TOL_Y
    dth, dX = g.gemm_backward(_cuda(th), Y, _cuda(dY))
    dto, dXo = oracle.backward(n, th, X64, dY.astype(np.float64))
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


def test_wide_angle_c3_sample(g):
    """C3 (n = 1024) in the bench launch configuration: 65536 columns with theta ~ U(-8 pi, 8 pi)
    plus special values; Y and dX on sampled columns vs the oracle, and dtheta of a 1024-column
    shard (every angle) vs the oracle's."""
    n, m = 1024, 65536
    th = _theta(n * (n - 1) // 2, "special", seed=31)
    X = synth.normal_matrix(n, m, seed=31, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=31, tid=synth.TID_DY)
    tt, Xt, dYt = _cuda(th), _cuda(X), _cuda(dY)
    Y = g.apply(tt, Xt)
    dth_full, dX = g.backward(tt, Y, dYt)
    cols = np.unique(np.concatenate([np.arange(4), np.random.default_rng(2).integers(0, m, 12), [m - 1]]))
    Xs, dYs = X[:, cols].astype(np.float64), dY[:, cols].astype(np.float64)
    assert rel(Y.cpu().numpy()[:, cols], oracle.apply(n, th, Xs)) <= TOL_Y
    _, dXo = oracle.backward(n, th, Xs, dYs)
    assert rel(dX.cpu().numpy()[:, cols], dXo) <= TOL_Y
    h = 1024
    d1, _ = g.backward(tt, Y[:, :h].contiguous(), dYt[:, :h].contiguous(), want_dX=False)
    dto, _ = oracle.backward(n, th, X[:, :h].astype(np.float64), dY[:, :h].astype(np.float64), want_dX=False)
    assert rel(d1.cpu().numpy(), dto) <= TOL_DTH
    assert np.isfinite(dth_full.cpu().numpy()).all()
