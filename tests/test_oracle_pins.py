"""Pins for the fp64 CPU oracle against what the paper and the mathematics fix.

Nothing here compares the oracle with itself: every expected value is a paper worked
example (tests/golden/, each cited), a closed form, an invariant, a library routine (numpy
LU determinant, dense matrix products of explicitly materialised G^e), brute force on tiny
inputs, or central finite differences.
"""
import os

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line)
    return rows


def _parse_pairs(line):
    return [tuple(int(v) for v in tok.split("-")) for tok in line.split()]


# ---------------------------------------------------------------- schedule (§3)

def test_schedule_eq5_n6():
    """Eq. (5): the n=6 round-robin sequence, verbatim and in order."""
    pairs, flat = oracle.schedule(6)
    want = [_parse_pairs(l) for l in _read_golden("eq5_n6_schedule.txt")]
    assert pairs.tolist() == [[list(p) for p in blk] for blk in want]
    assert flat.tolist() == [[3 * b + k for k in range(3)] for b in range(5)]


def test_fig1_sequences_give_eq5():
    """Fig. 1: pairing equal distances from the ends of each printed
    dimension sequence reproduces the oracle's blocks."""
    seqs = [[int(v) for v in l.split()] for l in _read_golden("fig1_n6_sequences.txt")]
    pairs, _ = oracle.schedule(6)
    for b, s in enumerate(seqs):
        blk = [tuple(sorted((s[k], s[5 - k]))) for k in range(3)]
        assert [tuple(p) for p in pairs[b].tolist()] == blk


def test_n4_Etilde_is_reversed_blocks():
    """E~ for n=4 is a round-robin sequence; it equals our n=4 blocks with the
    block order reversed (each pair sorted within its block as printed)."""
    et = _parse_pairs(_read_golden("n4_Etilde.txt")[0])
    pairs, _ = oracle.schedule(4)
    rev = [tuple(p) for blk in pairs[::-1].tolist() for p in blk]
    assert rev == et


def test_schedule_n2():
    pairs, flat = oracle.schedule(2)
    assert pairs.tolist() == [[[0, 1]]] and flat.tolist() == [[0]]


def _check_round_robin(n):
    pairs, flat = oracle.schedule(n)
    ne = n + (n % 2)
    R, S = ne - 1, ne // 2
    assert pairs.shape == (R, S, 2)
    i, j = pairs[..., 0].astype(np.int64), pairs[..., 1].astype(np.int64)
    assert (i < j).all()
    # every round a perfect matching of {0..ne-1} ("no two pairs share a coordinate")
    both = np.sort(np.concatenate([i, j], axis=1), axis=1)
    assert (both == np.arange(ne)[None, :]).all()
    # every pair exactly once ("each pair appears in exactly one block")
    code = (i * ne + j).ravel()
    assert np.unique(code).size == R * S == ne * (ne - 1) // 2
    # flat order: block-major over real pairs, bye pairs (j == n, odd n) have no angle
    real = j < n
    if n % 2:
        assert (real.sum(axis=1) == S - 1).all() and ((~real).sum(axis=1) == 1).all()
        assert (j[~real] == n).all()
    assert (flat[~real] == -1).all()
    assert (np.sort(flat[real].ravel()) == np.arange(n * (n - 1) // 2)).all()
    assert (flat[real].ravel() == np.arange(n * (n - 1) // 2)).all()  # block-major, listed order


@pytest.mark.parametrize("n", list(range(2, 130, 2)) + [256, 1024, 2048, 4096])
def test_schedule_even_round_robin(n):
    _check_round_robin(n)


@pytest.mark.parametrize("n", [3, 5, 7, 9, 15, 33, 127, 255, 1023, 2047])
def test_schedule_odd_bye(n):
    _check_round_robin(n)


def test_restriction_n8_m4():
    """n=8, m=4 removes exactly the 6 listed pairs, leaving 22."""
    lines = _read_golden("sec5_n8_m4_excluded.txt")
    excluded = set(_parse_pairs(lines[1]))
    E = oracle.sequence_E(8)
    mask = oracle.mask_from_keep(8, 4)
    got = {tuple(p) for p, k in zip(E.tolist(), mask) if not k}
    assert got == excluded and int(mask.sum()) == 22


@pytest.mark.parametrize("n,mk", [(8, 4), (9, 3), (16, 5), (33, 10), (64, 64), (64, 63), (10, 1)])
def test_restriction_count(n, mk):
    """N = m n - m(m+1)/2 free parameters (m = m_keep <= n-1; m_keep >= n-1 is
    unrestricted)."""
    mask = oracle.mask_from_keep(n, mk)
    mm = min(mk, n)
    assert int(mask.sum()) == mm * n - mm * (mm + 1) // 2


# ---------------------------------------------------------------- forward (§2-3)

def test_forward_n2_closed_form():
    """for n=2, U = G^{(0,1)} = [[cos, -sin], [sin, cos]]."""
    for th in [0.3, -2.5, 3.1, np.float32(np.pi / 2)]:
        th = np.float32(th)
        U = oracle.build_U(2, np.array([th], dtype=np.float32))
        c, s = np.cos(np.float64(th)), np.sin(np.float64(th))
        np.testing.assert_allclose(U, [[c, -s], [s, c]], rtol=0, atol=1e-15)


def test_rotate_rows_spec_examples():
    """Alg. 1 body: theta=pi/2 on I_2 -> [[0,-1],[1,0]]; (0,2) by pi/6 on I_3
    -> rows 0,2 = (sqrt3/2, 0, -1/2), (1/2, 0, sqrt3/2), row 1 untouched."""
    A = oracle.apply_sequence(2, np.array([[0, 1]]), np.array([np.pi / 2], np.float32), np.eye(2))
    np.testing.assert_allclose(A, [[0, -1], [1, 0]], atol=1e-7)
    th = np.float32(np.pi / 6)
    A = oracle.apply_sequence(3, np.array([[0, 2]]), np.array([th]), np.eye(3))
    c, s = np.cos(np.float64(th)), np.sin(np.float64(th))
    np.testing.assert_allclose(A, [[c, 0, -s], [0, 1, 0], [s, 0, c]], atol=1e-15)
    assert abs(c - np.sqrt(3) / 2) < 1e-7


@pytest.mark.parametrize("n", [2, 3, 4, 7, 16, 65])
def test_theta_zero_identity_bitwise(n):
    U = oracle.build_U(n, np.zeros(n * (n - 1) // 2, np.float32))
    assert (U == np.eye(n)).all()


@pytest.mark.parametrize("n", [4, 5, 16, 64, 256])
def test_orthogonal_det_plus_one(n):
    """U in SO(n): U^T U = I and det U = +1 (LAPACK LU via numpy)."""
    th = synth.theta(n * (n - 1) // 2, seed=n)
    U = oracle.build_U(n, th)
    assert np.abs(U.T @ U - np.eye(n)).max() <= 1e-12
    assert abs(np.linalg.det(U) - 1.0) <= 1e-9


def _dense_G(n, i, j, th):
    """G^e entries."""
    G = np.eye(n)
    c, s = np.cos(np.float64(th)), np.sin(np.float64(th))
    G[i, i] = G[j, j] = c
    G[i, j] = -s
    G[j, i] = s
    return G


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 8])
def test_forward_equals_dense_product(n):
    """Eq. (1): U = prod_{e in E} G^e(theta_e), E = circle-method sequence;
    brute-force dense products of the materialised G^e."""
    E = oracle.sequence_E(n)
    th = synth.theta(len(E), seed=10 + n)
    U = np.eye(n)
    for (i, j), t in zip(E.tolist(), th):
        U = U @ _dense_G(n, i, j, t)
    np.testing.assert_allclose(oracle.build_U(n, th), U, rtol=0, atol=1e-13)
    X = synth.normal_matrix(n, 7, seed=3, tid=synth.TID_X).astype(np.float64)
    np.testing.assert_allclose(oracle.apply(n, th, X), U @ X, rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.apply(n, th, X, transpose=True), U.T @ X, rtol=0, atol=1e-12)


def test_masked_forward_equals_dense_product_of_free():
    """§5 bypass: masked pairs are skipped == their G^e is the identity."""
    n = 8
    E = oracle.sequence_E(n)
    th = synth.theta(len(E), seed=5)
    mask = synth.random_mask(len(E), 0.6, seed=2)
    U = np.eye(n)
    for (i, j), t, k in zip(E.tolist(), th, mask):
        if k:
            U = U @ _dense_G(n, i, j, t)
    np.testing.assert_allclose(oracle.build_U(n, th, mask), U, rtol=0, atol=1e-13)
    th_nan = th.copy()
    th_nan[mask == 0] = np.nan
    assert (oracle.build_U(n, th_nan, mask) == oracle.build_U(n, th, mask)).all()


@pytest.mark.parametrize("n", [6, 32, 129])
def test_block_permutation_bitwise(n):
    """within a block the rotations act on disjoint rows and commute; any
    order of a block's pairs gives a bitwise-identical result (same fp64 operations per row)."""
    pairs, flat = oracle.schedule(n)
    E = oracle.sequence_E(n)
    th = synth.theta(len(E), seed=n)
    X = synth.normal_matrix(n, 5, seed=1, tid=synth.TID_X).astype(np.float64)
    ref = oracle.apply_sequence(n, E, th, X)
    rng = np.random.default_rng(n)
    order = []
    for b in range(pairs.shape[0]):
        idx = flat[b][flat[b] >= 0]
        order.extend(rng.permutation(idx).tolist())
    order = np.array(order)
    got = oracle.apply_sequence(n, E[order], th[order], X)
    assert (got == ref).all()


@pytest.mark.parametrize("n", [5, 64, 255])
def test_transpose_inverts_and_norms(n):
    th = synth.theta(n * (n - 1) // 2, seed=7)
    X = synth.normal_matrix(n, 9, seed=2, tid=synth.TID_X).astype(np.float64)
    Y = oracle.apply(n, th, X)
    np.testing.assert_allclose(np.linalg.norm(Y, axis=0), np.linalg.norm(X, axis=0), rtol=1e-13)
    np.testing.assert_allclose(oracle.apply(n, th, Y, transpose=True), X, rtol=0, atol=1e-12)


# ---------------------------------------------------------------- backward (§4)

def _fd_grad(n, th, X, dY, mask=None, h=1e-6):
    """Central finite differences of L = sum(dY * Y(theta)) (SPEC.md:267 recipe)."""
    g = np.zeros(th.size)
    th64 = th.astype(np.float64)
    for e in range(th.size):
        if mask is not None and not mask[e]:
            continue
        # perturb in fp64 through an explicit dense product (oracle takes fp32 theta)
        g[e] = (_loss_fd(n, th64, X, dY, e, h, mask) - _loss_fd(n, th64, X, dY, e, -h, mask)) / (2 * h)
    return g


def _loss_fd(n, th64, X, dY, e, h, mask):
    E = oracle.sequence_E(n)
    U = np.eye(n)
    for q, ((i, j), t) in enumerate(zip(E.tolist(), th64)):
        if mask is not None and not mask[q]:
            continue
        if q == e:
            t = t + h
        U = U @ _dense_G(n, i, j, t)
    return float(np.sum(dY * (U @ X)))


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 8])
def test_backward_finite_differences(n):
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=20 + n)
    X = synth.normal_matrix(n, 6, seed=4, tid=synth.TID_X).astype(np.float64)
    dY = synth.normal_matrix(n, 6, seed=4, tid=synth.TID_DY).astype(np.float64)
    dth, dX = oracle.backward(n, th, X, dY)
    fd = _fd_grad(n, th, X, dY)
    np.testing.assert_allclose(dth, fd, rtol=1e-6, atol=1e-7)
    # dX = U^T dY (chain rule of the linear map Y = U X), U by dense product
    np.testing.assert_allclose(dX, oracle.build_U(n, th).T @ dY, rtol=0, atol=1e-12)


def test_backward_restricted_fd_n8_m4():
    """SPEC.md:254 / PAPER.md:852-855: 22 free components match finite differences; the 6
    pinned ones are exactly 0."""
    n = 8
    mask = oracle.mask_from_keep(n, 4)
    th = synth.theta(28, seed=31)
    X = np.eye(n)
    dY = synth.normal_matrix(n, n, seed=5, tid=synth.TID_GAMMA).astype(np.float64)
    dth, _ = oracle.backward(n, th, X, dY, mask=mask)
    fd = _fd_grad(n, th, X, dY, mask=mask)
    np.testing.assert_allclose(dth, fd, rtol=1e-6, atol=1e-7)
    assert (dth[mask == 0] == 0).all() and (np.abs(dth[mask == 1]) > 0).sum() == 22


def _explicit_jacobian_vjp(n, th, Gamma):
    """dU/dtheta_e = U^{1:k-1} Q_e U^{k:n-1} with Q_e = -1 at (i,j), +1 at
    (j,i); contract with Gamma. Dense block products."""
    pairs, flat = oracle.schedule(n)
    R = pairs.shape[0]
    Gb = []
    for b in range(R):
        G = np.eye(n)
        for (i, j), f in zip(pairs[b].tolist(), flat[b]):
            if f >= 0:
                G = G @ _dense_G(n, i, j, th[f])
        Gb.append(G)
    out = np.zeros(th.size)
    cols = []
    for b in range(R):
        left = np.eye(n)
        for q in range(b):
            left = left @ Gb[q]
        right = np.eye(n)
        for q in range(b, R):
            right = right @ Gb[q]
        for (i, j), f in zip(pairs[b].tolist(), flat[b]):
            if f < 0:
                continue
            Q = np.zeros((n, n))
            Q[i, j] = -1.0
            Q[j, i] = 1.0
            J = left @ Q @ right
            cols.append(J)
            out[f] = np.sum(Gamma * J)
    return out, cols


@pytest.mark.parametrize("n", [3, 4, 6, 8])
def test_backward_explicit_jacobian_and_alg3(n):
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=40 + n)
    Gamma = synth.normal_matrix(n, n, seed=6, tid=synth.TID_GAMMA).astype(np.float64)
    want, cols = _explicit_jacobian_vjp(n, th, Gamma)
    dth, _ = oracle.backward(n, th, np.eye(n), Gamma)
    np.testing.assert_allclose(dth, want, rtol=0, atol=1e-10)
    # the paper's Algorithm 3 literally gives the same
    U = oracle.build_U(n, th)
    np.testing.assert_allclose(oracle.alg3(n, th, U, Gamma), want, rtol=0, atol=1e-10)
    # each Jacobian column has rank <= 2
    for J in cols:
        assert np.linalg.matrix_rank(J, tol=1e-9) <= 2


def test_backward_special_values():
    """n=2, theta=0, Gamma=[[0,0],[1,0]] -> dL/dtheta = cos 0 = 1; theta=0,
    Gamma=I -> 0 (Q_e has zero diagonal)."""
    dth, _ = oracle.backward(2, np.zeros(1, np.float32), np.eye(2), np.array([[0.0, 0.0], [1.0, 0.0]]))
    assert dth[0] == 1.0
    for n in [4, 7]:
        dth, _ = oracle.backward(n, np.zeros(n * (n - 1) // 2, np.float32), np.eye(n), np.eye(n))
        assert (dth == 0).all()


def test_backward_linear_in_dY():
    n = 16
    th = synth.theta(n * (n - 1) // 2, seed=3)
    X = synth.normal_matrix(n, 5, seed=1, tid=synth.TID_X).astype(np.float64)
    A = synth.normal_matrix(n, 5, seed=2, tid=synth.TID_DY).astype(np.float64)
    B = synth.normal_matrix(n, 5, seed=3, tid=synth.TID_DY).astype(np.float64)
    ga, xa = oracle.backward(n, th, X, A)
    gb, xb = oracle.backward(n, th, X, B)
    gc, xc = oracle.backward(n, th, X, 2.0 * A - 3.0 * B)
    np.testing.assert_allclose(gc, 2.0 * ga - 3.0 * gb, rtol=0, atol=1e-11)
    np.testing.assert_allclose(xc, 2.0 * xa - 3.0 * xb, rtol=0, atol=1e-12)


def test_backward_first_block_closed_form():
    """For e=(i,j) in b_1 (the last rotations applied), dL/dtheta_e = (Y dY^T - dY Y^T)_{ij}:
    Q_e structure with U^{1:0} = I."""
    n, m = 64, 33
    th = synth.theta(n * (n - 1) // 2, seed=9)
    X = synth.normal_matrix(n, m, seed=7, tid=synth.TID_X).astype(np.float64)
    dY = synth.normal_matrix(n, m, seed=7, tid=synth.TID_DY).astype(np.float64)
    Y = oracle.apply(n, th, X)
    dth, _ = oracle.backward(n, th, X, dY)
    pairs, flat = oracle.schedule(n)
    C = Y @ dY.T - dY @ Y.T
    for (i, j), f in zip(pairs[0].tolist(), flat[0]):
        assert abs(dth[f] - C[i, j]) <= 1e-10 * (1 + abs(C[i, j]))


def test_backward_masked_zero_and_nan():
    n = 9
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=11)
    mask = synth.random_mask(N, 0.5, seed=11)
    X = synth.normal_matrix(n, 4, seed=1, tid=synth.TID_X).astype(np.float64)
    dY = synth.normal_matrix(n, 4, seed=1, tid=synth.TID_DY).astype(np.float64)
    d1, x1 = oracle.backward(n, th, X, dY, mask=mask)
    th2 = th.copy()
    th2[mask == 0] = np.nan
    d2, x2 = oracle.backward(n, th2, X, dY, mask=mask)
    assert (d1[mask == 0] == 0).all()
    assert (d1 == d2).all() and (x1 == x2).all()
    fd = _fd_grad(n, th, X, dY, mask=mask)
    np.testing.assert_allclose(d1, fd, rtol=1e-6, atol=1e-7)
