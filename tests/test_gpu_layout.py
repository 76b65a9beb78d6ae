"""GPU parity for the layout options: circle-method start permutation
 and reflection, real and unitary, against the fp64
oracle with the same options, on every kernel family (register ring, idle-lane ring, multi-warp
ring, generic) and odd n (the bye moves with the permutation)."""
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


def _perm(n, seed):
    return np.random.default_rng(seed).permutation(n + n % 2).astype(np.int32)


# ring (8, 256, 1024), idle-lane (48, 1120), multi-warp (2047), generic (5, 100), odd (7, 33, 129)
LN = [2, 3, 5, 7, 8, 33, 48, 100, 129, 256, 1024, 1120, 2047]


@pytest.mark.parametrize("n", LN)
@pytest.mark.parametrize("variant", ["perm", "refl", "both"])
def test_layout_real_parity(g, n, variant):
    p = _perm(n, n) if variant in ("perm", "both") else None
    c = (n // 3) if variant in ("refl", "both") else None
    lay = g.Layout(n, perm=p, reflect_col=c)
    m = 37
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=n + 1)
    X = synth.normal_matrix(n, m, seed=n, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=n, tid=synth.TID_DY)
    tt, Xt = _cuda(th), _cuda(X)
    Y = g.apply(tt, Xt, layout=lay)
    assert rel(Y.cpu().numpy(), oracle.apply(n, th, X.astype(np.float64), perm=p, reflect=c)) <= TOL_Y
    Yt = g.apply(tt, Xt, transpose=True, layout=lay)
    assert rel(Yt.cpu().numpy(), oracle.apply(n, th, X.astype(np.float64), transpose=True, perm=p,
                                              reflect=c)) <= TOL_Y
    dth, dX = g.backward(tt, Y, _cuda(dY), layout=lay)
    dto, dXo = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64), perm=p, reflect=c)
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y
    if n <= 1024:
        U = g.build_U(tt, n, layout=lay).cpu().numpy()
        assert np.abs(U - oracle.build_U(n, th, perm=p, reflect=c)).max() <= 1e-5 * np.sqrt(n)


@pytest.mark.parametrize("n,mk", [(9, 3), (256, 100), (2047, 1024)])
def test_layout_masked_parity(g, n, mk):
    p = _perm(n, 3 * n)
    lay = g.Layout(n, perm=p, reflect_col=n - 1)
    mask = g.mask_from_keep(n, mk, perm=p)
    assert (mask == oracle.mask_from_keep(n, mk, perm=p)).all()
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=2)
    X = synth.normal_matrix(n, 20, seed=1, tid=synth.TID_X)
    dY = synth.normal_matrix(n, 20, seed=1, tid=synth.TID_DY)
    Y = g.apply(_cuda(th), _cuda(X), mask=_cuda(mask), layout=lay)
    assert rel(Y.cpu().numpy(), oracle.apply(n, th, X.astype(np.float64), mask, perm=p, reflect=n - 1)) <= TOL_Y
    dth, _ = g.backward(_cuda(th), Y, _cuda(dY), mask=_cuda(mask), want_dX=False, layout=lay)
    dto, _ = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64), mask, perm=p, reflect=n - 1)
    dth = dth.cpu().numpy()
    assert (dth[mask == 0] == 0).all()
    assert rel(dth, dto) <= TOL_DTH


@pytest.mark.parametrize("n", [3, 8, 48, 64, 256, 1023])
def test_layout_unitary_parity(g, n):
    p = _perm(n, 5 * n)
    c = n // 2
    lay = g.Layout(n, perm=p, reflect_col=c)
    N = n * (n - 1) // 2
    th, ph = synth.theta(N, seed=7), synth.theta(N, seed=8)
    m = 19
    X = (synth.normal_matrix(n, m, 1, synth.TID_X) + 1j * synth.normal_matrix(n, m, 2, synth.TID_X)).astype(np.complex64)
    G = (synth.normal_matrix(n, m, 1, synth.TID_DY) + 1j * synth.normal_matrix(n, m, 2, synth.TID_DY)).astype(np.complex64)
    tt, pt = _cuda(th), _cuda(ph)
    Y = g.u_apply(tt, pt, _cuda(X), layout=lay)
    Xd = X.astype(np.complex128)
    assert rel(Y.cpu().numpy(), oracle.u_apply(n, th, ph, Xd, perm=p, reflect=c)) <= TOL_Y
    Ya = g.u_apply(tt, pt, _cuda(X), adjoint=True, layout=lay)
    assert rel(Ya.cpu().numpy(), oracle.u_apply(n, th, ph, Xd, adjoint=True, perm=p, reflect=c)) <= TOL_Y
    dth, dph, dX = g.u_backward(tt, pt, Y, _cuda(G), layout=lay)
    dto, dpo, dXo = oracle.u_backward(n, th, ph, Xd, G.astype(np.complex128), perm=p, reflect=c)
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dph.cpu().numpy(), dpo) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


def test_layout_autograd_and_reuse(g):
    """GivensApply with a layout: the backward reuses the forward's tables (no recompute) and
    matches the oracle; det of the reflected U is -1."""
    n, m = 256, 64
    p = _perm(n, 1)
    lay = g.Layout(n, perm=p, reflect_col=17)
    th = synth.theta(n * (n - 1) // 2, seed=3)
    X = synth.normal_matrix(n, m, seed=3, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=3, tid=synth.TID_DY)
    tt = _cuda(th).requires_grad_(True)
    Xt = _cuda(X).requires_grad_(True)
    Y = g.givens_apply(tt, Xt, layout=lay)
    Y.backward(_cuda(dY))
    dto, dXo = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64), perm=p, reflect=17)
    assert rel(tt.grad.cpu().numpy(), dto) <= TOL_DTH
    assert rel(Xt.grad.cpu().numpy(), dXo) <= TOL_Y
    U = g.build_U(tt.detach(), n, layout=lay).double().cpu().numpy()
    sign, _ = np.linalg.slogdet(U)
    assert sign == -1.0
