"""Pins for the unitary (Appendix A) part of the fp64 oracle: U(n) membership, reduction to the
real path at phi = 0, closed forms, dense products of explicit G^e(theta, phi), the paper's Q_e /
P_e structure, and central finite differences of a real loss. None compares the oracle with
itself."""
import numpy as np
import pytest

import oracle
import synth


def _G(n, i, j, th, ph):
    """G^e(theta, phi) per Algorithm 4's row update: column i of the real
    Givens matrix times e^{i phi}."""
    G = np.eye(n, dtype=np.complex128)
    c, s = np.cos(np.float64(th)), np.sin(np.float64(th))
    e = np.exp(1j * np.float64(ph))
    G[i, i] = e * c
    G[j, j] = c
    G[i, j] = -s
    G[j, i] = e * s
    return G


def _dense_U(n, th, ph, mask=None):
    E = oracle.sequence_E(n)
    U = np.eye(n, dtype=np.complex128)
    for q, ((i, j), t, p) in enumerate(zip(E.tolist(), th, ph)):
        if mask is not None and not mask[q]:
            continue
        U = U @ _G(n, i, j, t, p)
    return U


def _cnormal(n, m, seed):
    return (synth.normal_matrix(n, m, seed, synth.TID_X).astype(np.float64)
            + 1j * synth.normal_matrix(n, m, seed, synth.TID_DY).astype(np.float64))


@pytest.mark.parametrize("n", [2, 3, 4, 7, 16, 64])
def test_unitary_membership(n):
    """U^dagger U = I (U(n)); |det U| = 1."""
    N = n * (n - 1) // 2
    U = oracle.u_build_U(n, synth.theta(N, seed=n), synth.theta(N, seed=n + 100))
    assert np.abs(U.conj().T @ U - np.eye(n)).max() <= 1e-12
    assert abs(abs(np.linalg.det(U)) - 1.0) <= 1e-9


@pytest.mark.parametrize("n", [5, 32])
def test_phi_zero_is_real_path_bitwise(n):
    """With all phases 0 the complex construction is the real one embedded."""
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=3)
    U = oracle.u_build_U(n, th, np.zeros(N, np.float32))
    assert (U.real == oracle.build_U(n, th)).all() and (U.imag == 0).all()


def test_n2_closed_forms():
    """n=2: U = G^{(0,1)} = [[e^{i phi} c, -s], [e^{i phi} s, c]]; theta=0, phi=pi -> diag(-1, 1)
    (SPEC.md:312)."""
    for th, ph in [(0.3, 1.1), (-2.0, 2.5), (0.0, np.pi)]:
        th, ph = np.float32(th), np.float32(ph)
        U = oracle.u_build_U(2, np.array([th]), np.array([ph]))
        e, c, s = np.exp(1j * np.float64(ph)), np.cos(np.float64(th)), np.sin(np.float64(th))
        np.testing.assert_allclose(U, [[e * c, -s], [e * s, c]], rtol=0, atol=1e-15)
    U = oracle.u_build_U(2, np.array([0.0], np.float32), np.array([np.pi], np.float32))
    np.testing.assert_allclose(U, [[-1, 0], [0, 1]], atol=1e-7)


@pytest.mark.parametrize("n", [3, 4, 6])
def test_dense_product_and_adjoint(n):
    N = n * (n - 1) // 2
    th, ph = synth.theta(N, seed=1), synth.theta(N, seed=2)
    mask = synth.random_mask(N, 0.7, seed=n)
    U = _dense_U(n, th, ph, mask)
    np.testing.assert_allclose(oracle.u_build_U(n, th, ph, mask), U, rtol=0, atol=1e-13)
    X = _cnormal(n, 5, 7)
    np.testing.assert_allclose(oracle.u_apply(n, th, ph, X, mask), U @ X, rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.u_apply(n, th, ph, X, mask, adjoint=True), U.conj().T @ X, rtol=0,
                               atol=1e-12)


def test_Q_and_P_structure():
    """Q_e = dG/dtheta G^dagger is -1 at (i,j), +1 at (j,i); P_e = dG/dphi G^dagger
    is i cos^2 at (i,i), i sin^2 at (j,j), i sin cos at (i,j) and (j,i). Holds for Alg. 4's G (phase
    on column i only) -- pins reading R15."""
    n, i, j = 4, 1, 3
    th, ph, h = 0.7, -1.3, 1e-6
    G = _G(n, i, j, th, ph)
    dGt = (_G(n, i, j, th + h, ph) - _G(n, i, j, th - h, ph)) / (2 * h)
    dGp = (_G(n, i, j, th, ph + h) - _G(n, i, j, th, ph - h)) / (2 * h)
    Q = dGt @ G.conj().T
    P = dGp @ G.conj().T
    Qw = np.zeros((n, n), complex); Qw[i, j] = -1; Qw[j, i] = 1
    c, s = np.cos(th), np.sin(th)
    Pw = np.zeros((n, n), complex)
    Pw[i, i], Pw[j, j], Pw[i, j], Pw[j, i] = 1j * c * c, 1j * s * s, 1j * s * c, 1j * s * c
    np.testing.assert_allclose(Q, Qw, atol=1e-8)
    np.testing.assert_allclose(P, Pw, atol=1e-8)


def _loss(U, X, Gam):
    """Real loss whose gradient w.r.t. Y = U X is Gam under Gamma = dL/dRe + i dL/dIm."""
    Y = U @ X
    return float(np.sum(Gam.real * Y.real + Gam.imag * Y.imag))


@pytest.mark.parametrize("n", [2, 3, 5, 6])
def test_unitary_backward_finite_differences(n):
    N = n * (n - 1) // 2
    th, ph = synth.theta(N, seed=11), synth.theta(N, seed=12)
    X, Gam = _cnormal(n, 4, 1), _cnormal(n, 4, 2)
    dth, dph, dX = oracle.u_backward(n, th, ph, X, Gam)
    th64, ph64 = th.astype(np.float64), ph.astype(np.float64)
    h = 1e-6
    E = oracle.sequence_E(n)

    def U_of(t, p):
        U = np.eye(n, dtype=np.complex128)
        for (i, j), a, b in zip(E.tolist(), t, p):
            U = U @ _G(n, i, j, a, b)
        return U

    for e in range(N):
        tp, tm = th64.copy(), th64.copy()
        tp[e] += h; tm[e] -= h
        fd = (_loss(U_of(tp, ph64), X, Gam) - _loss(U_of(tm, ph64), X, Gam)) / (2 * h)
        assert abs(dth[e] - fd) <= 1e-6 * (1 + abs(fd))
        pp, pm = ph64.copy(), ph64.copy()
        pp[e] += h; pm[e] -= h
        fd = (_loss(U_of(th64, pp), X, Gam) - _loss(U_of(th64, pm), X, Gam)) / (2 * h)
        assert abs(dph[e] - fd) <= 1e-6 * (1 + abs(fd))
    # dX = U^dagger Gamma (adjoint of the linear map under the real-pair convention)
    np.testing.assert_allclose(dX, U_of(th64, ph64).conj().T @ Gam, rtol=0, atol=1e-12)


def test_unitary_jacobian_ranks():
    """dU/dtheta_e has rank <= 2, dU/dphi_e has rank 1 (via the explicit
    products U^{1:k-1} Q_e U^{k:n-1} and U^{1:k-1} P_e U^{k:n-1}, dense)."""
    n = 6
    N = n * (n - 1) // 2
    th, ph = synth.theta(N, seed=5), synth.theta(N, seed=6)
    pairs, flat = oracle.schedule(n)
    Gb = []
    for b in range(pairs.shape[0]):
        G = np.eye(n, dtype=complex)
        for (i, j), f in zip(pairs[b].tolist(), flat[b]):
            G = G @ _G(n, i, j, th[f], ph[f])
        Gb.append(G)
    for b in range(pairs.shape[0]):
        left = np.eye(n, dtype=complex)
        for q in range(b):
            left = left @ Gb[q]
        right = np.eye(n, dtype=complex)
        for q in range(b, len(Gb)):
            right = right @ Gb[q]
        for (i, j), f in zip(pairs[b].tolist(), flat[b]):
            c, s = np.cos(np.float64(th[f])), np.sin(np.float64(th[f]))
            Q = np.zeros((n, n), complex); Q[i, j] = -1; Q[j, i] = 1
            P = np.zeros((n, n), complex)
            P[i, i], P[j, j], P[i, j], P[j, i] = 1j * c * c, 1j * s * s, 1j * s * c, 1j * s * c
            assert np.linalg.matrix_rank(left @ Q @ right, tol=1e-9) <= 2
            assert np.linalg.matrix_rank(left @ P @ right, tol=1e-9) == 1


def test_unitary_special_values_and_mask():
    """theta=phi=0, Gamma=I -> dtheta = dphi = 0 on a real identity Gamma;
    n=2, Gamma=[[i,0],[0,0]] -> dphi = 1. Masked angles: exactly 0."""
    for n in [2, 5]:
        N = n * (n - 1) // 2
        dth, dph, _ = oracle.u_backward(n, np.zeros(N, np.float32), np.zeros(N, np.float32),
                                        np.eye(n, dtype=complex), np.eye(n, dtype=complex))
        assert (dth == 0).all() and (np.abs(dph) == 0).all()
    dth, dph, _ = oracle.u_backward(2, np.zeros(1, np.float32), np.zeros(1, np.float32), np.eye(2, dtype=complex),
                                    np.array([[1j, 0], [0, 0]]))
    assert dth[0] == 0 and abs(dph[0] - 1.0) < 1e-15
    n = 7
    N = n * (n - 1) // 2
    mask = synth.random_mask(N, 0.5, seed=1)
    dth, dph, _ = oracle.u_backward(n, synth.theta(N, 1), synth.theta(N, 2), _cnormal(n, 3, 1), _cnormal(n, 3, 2),
                                    mask=mask)
    assert (dth[mask == 0] == 0).all() and (dph[mask == 0] == 0).all()
