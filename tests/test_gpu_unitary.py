"""GPU parity for the unitary U(n) variant (Appendix A, Algorithm 4; readings R15/R16):
the sm_100a path through the C ABI against the fp64 oracle (oracle.u_apply / u_backward) on the
same seeded inputs. Complex tolerances are the real ones of BASELINE.json north_star applied to the
complex norms: ||dY||/||Y|| <= 1e-5, ||d dtheta||/||dtheta|| and ||d dphi||/||dphi|| <= 1e-4,
max|dU| <= 1e-5 sqrt(n)."""
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




def _c(n, m, seed, tid):
    return (synth.normal_matrix(n, m, seed, tid).astype(np.float64)
            + 1j * synth.normal_matrix(n, m, seed + 7919, tid).astype(np.float64))


def _inputs(n, m, seed=0, mask_keep=None, mask_p=None):
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=seed)
    ph = synth.theta(N, seed=seed + 1)
    X = _c(n, m, seed, synth.TID_X)
    G = _c(n, m, seed, synth.TID_DY)
    mask = None
    if mask_keep is not None:
        mask = oracle.mask_from_keep(n, mask_keep)
    elif mask_p is not None:
        mask = synth.random_mask(N, mask_p, seed=seed)
    return th, ph, X, G, mask


def _cuda(a):
    if a is None:
        return None
    if np.iscomplexobj(a):
        a = a.astype(np.complex64)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ring configurations (8, 16, 32, 128, 256, 512, 1024, 2047), idle-lane rings (48, 96, 1120, 63/64:
# the W = 32 ring replaced by W = 16 with idle lanes) and the generic kernel (2..7, 9, 17, 33, 65,
# 100, 300, 4096)
U_N = [2, 3, 4, 5, 6, 7, 8, 9, 16, 17, 32, 33, 48, 63, 64, 65, 96, 100, 128, 256, 300, 511, 512, 768, 1023,
       1024, 1120, 2047]


@pytest.mark.parametrize("n", U_N)
@pytest.mark.parametrize("m", [1, 19, 130])
def test_u_apply_parity(g, n, m):
    th, ph, X, _, _ = _inputs(n, m, seed=n + m)
    Y = g.u_apply(_cuda(th), _cuda(ph), _cuda(X)).cpu().numpy()
    assert rel(Y, oracle.u_apply(n, th, ph, X)) <= TOL_Y
    Ya = g.u_apply(_cuda(th), _cuda(ph), _cuda(X), adjoint=True).cpu().numpy()
    assert rel(Ya, oracle.u_apply(n, th, ph, X, adjoint=True)) <= TOL_Y


@pytest.mark.parametrize("n", U_N)
@pytest.mark.parametrize("m", [1, 23, 129])
def test_u_backward_parity(g, n, m):
    th, ph, X, G, _ = _inputs(n, m, seed=3 * n + m)
    dto, dpo, dXo = oracle.u_backward(n, th, ph, X, G)
    Y = g.u_apply(_cuda(th), _cuda(ph), _cuda(X))
    dth, dph, dX = g.u_backward(_cuda(th), _cuda(ph), Y, _cuda(G))
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dph.cpu().numpy(), dpo) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


@pytest.mark.parametrize("n", [2, 3, 8, 33, 64, 256, 1024, 2047, 2048])
def test_u_build_U_parity_and_unitarity(g, n):
    N = n * (n - 1) // 2
    th, ph = synth.theta(N, seed=21), synth.theta(N, seed=22)
    U = g.u_build_U(_cuda(th), _cuda(ph), n).cpu().numpy().astype(np.complex128)
    assert np.abs(U - oracle.u_build_U(n, th, ph)).max() <= 1e-5 * np.sqrt(n)
    assert np.abs(U.conj().T @ U - np.eye(n)).max() <= 1e-5 * np.sqrt(n)


def test_u_generic_large_n(g):
    """n = 4096 (S = 2048) has no unitary ring: the generic kernel, at a few columns."""
    n, m = 4096, 3
    th, ph, X, G, _ = _inputs(n, m, seed=5)
    Y = g.u_apply(_cuda(th), _cuda(ph), _cuda(X))
    assert rel(Y.cpu().numpy(), oracle.u_apply(n, th, ph, X)) <= TOL_Y
    dto, dpo, dXo = oracle.u_backward(n, th, ph, X, G)
    dth, dph, dX = g.u_backward(_cuda(th), _cuda(ph), Y, _cuda(G))
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dph.cpu().numpy(), dpo) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


@pytest.mark.parametrize("n,mk", [(8, 4), (9, 3), (64, 20), (256, 100), (1024, 512), (2047, 1024)])
def test_u_restricted_parity(g, n, mk):
    """Paper §5 restriction applied to the unitary variant: masked angles are identities and get
    exactly zero dtheta and dphi."""
    th, ph, X, G, mask = _inputs(n, 33, seed=n, mask_keep=mk)
    Y = g.u_apply(_cuda(th), _cuda(ph), _cuda(X), mask=_cuda(mask))
    assert rel(Y.cpu().numpy(), oracle.u_apply(n, th, ph, X, mask)) <= TOL_Y
    dto, dpo, dXo = oracle.u_backward(n, th, ph, X, G, mask)
    dth, dph, dX = g.u_backward(_cuda(th), _cuda(ph), Y, _cuda(G), mask=_cuda(mask))
    dth, dph = dth.cpu().numpy(), dph.cpu().numpy()
    assert (dth[mask == 0] == 0).all() and (dph[mask == 0] == 0).all()
    assert rel(dth, dto) <= TOL_DTH and rel(dph, dpo) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


@pytest.mark.parametrize("n", [7, 256])
def test_u_random_mask_parity(g, n):
    th, ph, X, G, mask = _inputs(n, 40, seed=2 * n, mask_p=0.6)
    Y = g.u_apply(_cuda(th), _cuda(ph), _cuda(X), mask=_cuda(mask))
    assert rel(Y.cpu().numpy(), oracle.u_apply(n, th, ph, X, mask)) <= TOL_Y
    dto, dpo, _ = oracle.u_backward(n, th, ph, X, G, mask)
    dth, dph, _ = g.u_backward(_cuda(th), _cuda(ph), Y, _cuda(G), mask=_cuda(mask), want_dX=False)
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH and rel(dph.cpu().numpy(), dpo) <= TOL_DTH


def test_u_phi_zero_matches_real_path(g):
    """phi = 0 reduces G^e to the real rotation: the unitary kernels on X = A + iB
    give apply(A) + i apply(B) of the real kernels, and dtheta the sum of the two real dthetas."""
    n, m = 256, 64
    N = n * (n - 1) // 2
    th = _cuda(synth.theta(N, seed=9))
    zero = torch.zeros(N, device="cuda")
    A = _cuda(synth.normal_matrix(n, m, 1, synth.TID_X))
    B = _cuda(synth.normal_matrix(n, m, 2, synth.TID_X))
    Y = g.u_apply(th, zero, torch.complex(A, B))
    YA, YB = g.apply(th, A), g.apply(th, B)
    torch.testing.assert_close(Y.real, YA, rtol=0, atol=1e-5)
    torch.testing.assert_close(Y.imag, YB, rtol=0, atol=1e-5)
    dA = _cuda(synth.normal_matrix(n, m, 3, synth.TID_DY))
    dB = _cuda(synth.normal_matrix(n, m, 4, synth.TID_DY))
    dth, _, dX = g.u_backward(th, zero, Y, torch.complex(dA, dB))
    tA, xA = g.backward(th, YA, dA)
    tB, xB = g.backward(th, YB, dB)
    ref = (tA + tB).cpu().numpy()
    assert rel(dth.cpu().numpy(), ref) <= 1e-5
    torch.testing.assert_close(dX.real, xA, rtol=0, atol=1e-5)
    torch.testing.assert_close(dX.imag, xB, rtol=0, atol=1e-5)


def test_u_determinism_and_strided(g):
    n, m = 512, 300
    th, ph, X, G, _ = _inputs(n, m, seed=4)
    tt, pt = _cuda(th), _cuda(ph)
    Xt = _cuda(X)
    Y1 = g.u_apply(tt, pt, Xt)
    a = g.u_backward(tt, pt, Y1, _cuda(G))
    b = g.u_backward(tt, pt, Y1, _cuda(G))
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    # strided leading dimension: a column window of a wider matrix
    big = torch.zeros((n, m + 17), dtype=torch.complex64, device="cuda")
    big[:, 5:5 + m] = Xt
    Xv = big[:, 5:5 + m]
    out = torch.full((n, m + 9), 7 + 7j, dtype=torch.complex64, device="cuda")
    g.u_apply(tt, pt, Xv, out=out[:, 2:2 + m])
    assert torch.equal(out[:, 2:2 + m], Y1)
    assert (out[:, :2] == 7 + 7j).all() and (out[:, 2 + m:] == 7 + 7j).all()


def test_u_medium_full_parity(g):
    """n = 1024 at 2048 complex columns (~64 ring slabs per CTA pass): every output element."""
    n, m = 1024, 2048
    th, ph, X, G, _ = _inputs(n, m, seed=77)
    Y = g.u_apply(_cuda(th), _cuda(ph), _cuda(X))
    assert rel(Y.cpu().numpy(), oracle.u_apply(n, th, ph, X)) <= TOL_Y
    dto, dpo, dXo = oracle.u_backward(n, th, ph, X, G)
    dth, dph, dX = g.u_backward(_cuda(th), _cuda(ph), Y, _cuda(G))
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dph.cpu().numpy(), dpo) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


def test_u_bad_arguments(g):
    th = torch.zeros(6, device="cuda")
    X = torch.zeros((4, 3), dtype=torch.complex64, device="cuda")
    with pytest.raises(ValueError):
        g.u_apply(th, torch.zeros(5, device="cuda"), X)  # phi of the wrong length
    with pytest.raises(ValueError):
        g.u_apply(th, th, X.real.contiguous())  # not complex
    assert not g.u_supported(1) and g.u_supported(2) and g.u_supported(4096)
