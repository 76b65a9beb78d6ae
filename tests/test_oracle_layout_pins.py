"""Pins for the oracle's layout options: the circle method's initial
permutation ("could have been arbitrarily permuted") and the
reflection class (det -1 "by for example negating an arbitrary fixed column
following the construction"). Expected values are hand traces of the circle method, relabelings
of the identity schedule, dense products of explicit G^e, LAPACK determinants and finite
differences -- never the oracle compared with itself."""
import numpy as np
import pytest

import oracle
import synth


def _perm(n, seed):
    ne = n + (n % 2)
    return np.random.default_rng(seed).permutation(ne).astype(np.int32)


def _dense_G(n, i, j, th):
    G = np.eye(n)
    c, s = np.cos(np.float64(th)), np.sin(np.float64(th))
    G[i, i] = G[j, j] = c
    G[i, j] = -s
    G[j, i] = s
    return G


def _dense_U(n, E, th, mask=None):
    U = np.eye(n)
    for q, ((i, j), t) in enumerate(zip(E.tolist(), th)):
        if mask is None or mask[q]:
            U = U @ _dense_G(n, i, j, t)
    return U


def test_n4_permuted_hand_trace():
    """Circle method from (3, 1, 0, 2) (PAPER.md:371-377 by hand): pair equal distances from the
    ends, hold the first element, rotate the rest right by one: (3,1,0,2) -> (3,2,1,0) -> (3,0,2,1)."""
    pairs, flat = oracle.schedule(4, perm=[3, 1, 0, 2])
    assert pairs.tolist() == [[[2, 3], [0, 1]], [[0, 3], [1, 2]], [[1, 3], [0, 2]]]
    assert flat.tolist() == [[0, 1], [2, 3], [4, 5]]


def test_n3_permuted_bye_hand_trace():
    """Odd n: the bye index n = 3 is part of the permuted sequence; from (1, 3, 0, 2):
    (1,3,0,2) -> (1,2,3,0) -> (1,0,2,3); pairs containing 3 are byes (no angle)."""
    pairs, flat = oracle.schedule(3, perm=[1, 3, 0, 2])
    assert pairs.tolist() == [[[1, 2], [0, 3]], [[0, 1], [2, 3]], [[1, 3], [0, 2]]]
    assert flat.tolist() == [[0, -1], [1, -1], [-1, 2]]


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 9, 16, 31, 64, 65])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_permuted_schedule_is_relabeled_identity(n, seed):
    """The circle method acts on sequence positions, so starting from perm relabels every pair of
    the identity schedule through perm (then sorts it); still a round-robin (perfect matchings,
    exact cover) with one bye per round for odd n and the block-major flat order."""
    p = _perm(n, seed)
    ne = len(p)
    pairs, flat = oracle.schedule(n, perm=p)
    pid, _ = oracle.schedule(n)
    want = np.sort(p[pid], axis=-1)
    assert (pairs == want).all()
    i, j = pairs[..., 0].astype(np.int64), pairs[..., 1].astype(np.int64)
    both = np.sort(np.concatenate([i, j], axis=1), axis=1)
    assert (both == np.arange(ne)[None, :]).all()
    assert np.unique((i * ne + j).ravel()).size == ne * (ne - 1) // 2
    real = j < n
    assert (flat[~real] == -1).all()
    assert (flat[real].ravel() == np.arange(n * (n - 1) // 2)).all()


def test_identity_perm_is_default_and_bad_perm_rejected():
    for n in [6, 7]:
        ne = n + n % 2
        a, fa = oracle.schedule(n)
        b, fb = oracle.schedule(n, perm=np.arange(ne))
        assert (a == b).all() and (fa == fb).all()
    with pytest.raises(ValueError):
        oracle.schedule(6, perm=[0, 1, 2, 3, 4, 4])
    with pytest.raises(ValueError):
        oracle.schedule(6, perm=[0, 1, 2, 3, 4, 6])


@pytest.mark.parametrize("n", [3, 4, 5, 6, 8])
def test_permuted_forward_equals_dense_product(n):
    p = _perm(n, n)
    E = oracle.sequence_E(n, p)
    th = synth.theta(len(E), seed=30 + n)
    U = _dense_U(n, E, th)
    np.testing.assert_allclose(oracle.build_U(n, th, perm=p), U, rtol=0, atol=1e-13)
    X = synth.normal_matrix(n, 5, seed=3, tid=synth.TID_X).astype(np.float64)
    np.testing.assert_allclose(oracle.apply(n, th, X, perm=p), U @ X, rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.apply(n, th, X, perm=p, transpose=True), U.T @ X, rtol=0, atol=1e-12)
    assert abs(np.linalg.det(U) - 1) < 1e-9


def test_reflection_spec_example():
    """n=4, all theta = 0, reflect column 0 -> diag(-1, 1, 1, 1), det -1."""
    U = oracle.build_U(4, np.zeros(6, np.float32), reflect=0)
    assert (U == np.diag([-1.0, 1, 1, 1])).all()
    assert np.linalg.det(U) == pytest.approx(-1.0)


@pytest.mark.parametrize("n,c", [(2, 1), (5, 0), (16, 7), (65, 64)])
def test_reflection_negates_a_column(n, c):
    """U' = U with column c negated, bitwise (negation is exact and the
    rotation arithmetic is sign-symmetric); det U' = -1; apply/transpose are U' X and U'^T X."""
    th = synth.theta(n * (n - 1) // 2, seed=n)
    U = oracle.build_U(n, th)
    Ur = oracle.build_U(n, th, reflect=c)
    Uneg = U.copy()
    Uneg[:, c] = -Uneg[:, c]
    assert (Ur == Uneg).all()
    assert np.linalg.det(Ur) == pytest.approx(-1.0, abs=1e-9)
    X = synth.normal_matrix(n, 4, seed=1, tid=synth.TID_X).astype(np.float64)
    np.testing.assert_allclose(oracle.apply(n, th, X, reflect=c), Uneg @ X, rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.apply(n, th, X, reflect=c, transpose=True), Uneg.T @ X, rtol=0, atol=1e-12)


@pytest.mark.parametrize("n", [3, 4, 5, 6])
def test_backward_fd_with_perm_and_reflection(n):
    p = _perm(n, 7 * n)
    c = n // 2
    E = oracle.sequence_E(n, p)
    N = len(E)
    th = synth.theta(N, seed=40 + n)
    X = synth.normal_matrix(n, 5, seed=5, tid=synth.TID_X).astype(np.float64)
    dY = synth.normal_matrix(n, 5, seed=5, tid=synth.TID_DY).astype(np.float64)
    dth, dX = oracle.backward(n, th, X, dY, perm=p, reflect=c)
    D = np.eye(n)
    D[c, c] = -1
    th64 = th.astype(np.float64)
    h = 1e-6
    for e in range(N):
        tp, tm = th64.copy(), th64.copy()
        tp[e] += h
        tm[e] -= h
        fd = (np.sum(dY * (_dense_U(n, E, tp) @ D @ X)) - np.sum(dY * (_dense_U(n, E, tm) @ D @ X))) / (2 * h)
        assert abs(dth[e] - fd) <= 1e-6 * (1 + abs(fd))
    np.testing.assert_allclose(dX, (_dense_U(n, E, th64) @ D).T @ dY, rtol=0, atol=1e-12)


def test_alg3_with_perm_equals_fd():
    """Algorithm 3 literally on the permuted sequence == finite differences of
    <Gamma, U(theta)>."""
    n = 6
    p = _perm(n, 3)
    E = oracle.sequence_E(n, p)
    th = synth.theta(len(E), seed=2)
    Gam = synth.normal_matrix(n, n, seed=9, tid=synth.TID_GAMMA).astype(np.float64)
    U = oracle.build_U(n, th, perm=p)
    d = oracle.alg3(n, th, U, Gam, perm=p)
    th64 = th.astype(np.float64)
    for e in range(len(E)):
        tp, tm = th64.copy(), th64.copy()
        tp[e] += 1e-6
        tm[e] -= 1e-6
        fd = (np.sum(Gam * _dense_U(n, E, tp)) - np.sum(Gam * _dense_U(n, E, tm))) / 2e-6
        assert abs(d[e] - fd) <= 1e-6 * (1 + abs(fd))


def test_restriction_under_perm():
    """§5: the excluded set depends only on the pairs, so the count
    m_keep n - m_keep (m_keep + 1) / 2 holds for any start permutation."""
    for n, mk in [(8, 4), (9, 3), (33, 10)]:
        mask = oracle.mask_from_keep(n, mk, perm=_perm(n, n + mk))
        assert int(mask.sum()) == mk * n - mk * (mk + 1) // 2


def _G_u(n, i, j, th, ph):
    G = np.eye(n, dtype=complex)
    c, s, e = np.cos(np.float64(th)), np.sin(np.float64(th)), np.exp(1j * np.float64(ph))
    G[i, i], G[j, j], G[i, j], G[j, i] = e * c, c, -s, e * s
    return G


@pytest.mark.parametrize("n", [3, 4, 6])
def test_unitary_perm_and_reflection_dense(n):
    p = _perm(n, 11 * n)
    c = 1
    E = oracle.sequence_E(n, p)
    th, ph = synth.theta(len(E), seed=1), synth.theta(len(E), seed=2)
    U = np.eye(n, dtype=complex)
    for (i, j), t, f in zip(E.tolist(), th, ph):
        U = U @ _G_u(n, i, j, t, f)
    U[:, c] = -U[:, c]
    np.testing.assert_allclose(oracle.u_build_U(n, th, ph, perm=p, reflect=c), U, rtol=0, atol=1e-13)
    X = (synth.normal_matrix(n, 3, 1, synth.TID_X) + 1j * synth.normal_matrix(n, 3, 2, synth.TID_X)).astype(complex)
    np.testing.assert_allclose(oracle.u_apply(n, th, ph, X, perm=p, reflect=c), U @ X, rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.u_apply(n, th, ph, X, perm=p, reflect=c, adjoint=True), U.conj().T @ X,
                               rtol=0, atol=1e-12)
    Gam = (synth.normal_matrix(n, 3, 3, synth.TID_DY) + 1j * synth.normal_matrix(n, 3, 4, synth.TID_DY)).astype(complex)
    dth, dph, dX = oracle.u_backward(n, th, ph, X, Gam, perm=p, reflect=c)
    np.testing.assert_allclose(dX, U.conj().T @ Gam, rtol=0, atol=1e-12)
    # finite differences of L = Re<Gam, U X> (reading R16) for theta and phi
    th64, ph64 = th.astype(np.float64), ph.astype(np.float64)

    def L(t, f):
        V = np.eye(n, dtype=complex)
        for (i, j), a, b in zip(E.tolist(), t, f):
            V = V @ _G_u(n, i, j, a, b)
        V[:, c] = -V[:, c]
        Y = V @ X
        return float(np.sum(Gam.real * Y.real + Gam.imag * Y.imag))

    for e in range(len(E)):
        for arr, got in ((0, dth), (1, dph)):
            a, b = [th64.copy(), ph64.copy()], [th64.copy(), ph64.copy()]
            a[arr][e] += 1e-6
            b[arr][e] -= 1e-6
            fd = (L(*a) - L(*b)) / 2e-6
            assert abs(got[e] - fd) <= 1e-6 * (1 + abs(fd))
