"""GPU parity: the sm_100a path (through the C ABI) against the fp64 CPU oracle on the same
seeded inputs, element by element.

Tolerances (BASELINE.json north_star): schedule/indexing bit-exact; fp32
max|dU| <= 1e-5 sqrt(n), ||dY||/||Y|| <= 1e-5, ||d dtheta||/||dtheta|| <= 1e-4; dX uses the
Y bound (reading R13)."""
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




def _inputs(n, m, seed=0, mask_keep=None, mask_p=None):
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=seed)
    X = synth.normal_matrix(n, m, seed=seed, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=seed, tid=synth.TID_DY)
    mask = None
    if mask_keep is not None:
        mask = oracle.mask_from_keep(n, mask_keep)
    elif mask_p is not None:
        mask = synth.random_mask(N, mask_p, seed=seed)
    return th, X, dY, mask


def _cuda(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


ALL_N = [2, 3, 4, 5, 6, 7, 8, 9, 12, 15, 16, 17, 31, 32, 33, 48, 63, 64, 65, 96, 100, 127, 128, 129, 160, 255,
         256, 300, 511, 512, 768, 1023, 1024, 1120, 2047, 2048]
# ring configurations with idle lanes (S = W * La, La not a power of two): 48, 96, 160, 768, 1120,
# and below 1535, 2000 (W=8, La=125 of 128), 2400 (a fully idle trailing warp)


@pytest.mark.parametrize("n", ALL_N + [1535, 2000, 2400, 4096])
@pytest.mark.parametrize("direction", [0, 1])
def test_index_trace_bit_exact(g, n, direction):
    """The kernels' on-device data movement pairs exactly the schedule's rows (bit-exact)."""
    got = g.index_trace(n, direction).cpu().numpy()
    pairs, _ = oracle.schedule(n)
    assert (got == pairs).all()


@pytest.mark.parametrize("n", ALL_N)
@pytest.mark.parametrize("m", [1, 37, 300])
def test_apply_parity(g, n, m):
    th, X, _, _ = _inputs(n, m, seed=n + m)
    Y = g.apply(_cuda(th), _cuda(X)).cpu().numpy()
    Yo = oracle.apply(n, th, X.astype(np.float64))
    assert rel(Y, Yo) <= TOL_Y
    Yt = g.apply(_cuda(th), _cuda(X), transpose=True).cpu().numpy()
    Yto = oracle.apply(n, th, X.astype(np.float64), transpose=True)
    assert rel(Yt, Yto) <= TOL_Y


@pytest.mark.parametrize("n", [2, 3, 6, 8, 16, 33, 64, 256, 1024, 2047, 4096])
def test_build_U_parity(g, n):
    th = synth.theta(n * (n - 1) // 2, seed=5)
    U = g.build_U(_cuda(th), n).cpu().numpy()
    Uo = oracle.build_U(n, th)
    assert np.abs(U - Uo).max() <= 1e-5 * np.sqrt(n)


@pytest.mark.parametrize("n", ALL_N)
@pytest.mark.parametrize("m", [1, 45, 257])
def test_backward_parity(g, n, m):
    th, X, dY, _ = _inputs(n, m, seed=3 * n + m)
    tt, Xt, dYt = _cuda(th), _cuda(X), _cuda(dY)
    Y = g.apply(tt, Xt)
    dth, dX = g.backward(tt, Y, dYt)
    dto, dXo = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64))
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


@pytest.mark.parametrize("n,mk", [(8, 4), (9, 3), (64, 20), (256, 100), (1024, 512), (2047, 1024)])
def test_restricted_parity(g, n, mk):
    """§5 restriction: pinned angles bypassed, their dtheta exactly 0, and a
    NaN in a pinned theta has no effect."""
    m = 70
    th, X, dY, mask = _inputs(n, m, seed=n, mask_keep=mk)
    th_nan = th.copy()
    th_nan[mask == 0] = np.nan
    tt, Xt, dYt, mt = _cuda(th_nan), _cuda(X), _cuda(dY), _cuda(mask)
    Y = g.apply(tt, Xt, mask=mt)
    dth, dX = g.backward(tt, Y, dYt, mask=mt)
    Yo = oracle.apply(n, th, X.astype(np.float64), mask=mask)
    dto, dXo = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64), mask=mask)
    d = dth.cpu().numpy()
    assert rel(Y.cpu().numpy(), Yo) <= TOL_Y
    assert (d[mask == 0] == 0).all()
    assert rel(d, dto) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y


@pytest.mark.parametrize("n", [7, 256])
def test_random_mask_parity(g, n):
    m = 50
    th, X, dY, mask = _inputs(n, m, seed=9, mask_p=0.5)
    tt, Xt, dYt, mt = _cuda(th), _cuda(X), _cuda(dY), _cuda(mask)
    Y = g.apply(tt, Xt, mask=mt)
    dth, dX = g.backward(tt, Y, dYt, mask=mt)
    dto, dXo = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64), mask=mask)
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert (dth.cpu().numpy()[mask == 0] == 0).all()


def test_u_backward_is_alg3(g):
    """U-build gradient: givens_backward(Y=U, dY=Gamma) equals the paper's Algorithm 3."""
    n = 64
    th = synth.theta(n * (n - 1) // 2, seed=2)
    Gm = synth.normal_matrix(n, n, seed=2, tid=synth.TID_GAMMA)
    U = g.build_U(_cuda(th), n)
    dth, _ = g.backward(_cuda(th), U, _cuda(Gm), want_dX=False)
    want = oracle.alg3(n, th, oracle.build_U(n, th), Gm.astype(np.float64))
    assert rel(dth.cpu().numpy(), want) <= TOL_DTH


def test_theta_zero_identity_bitwise(g):
    for n in [8, 64, 1024]:
        U = g.build_U(torch.zeros(n * (n - 1) // 2, device="cuda"), n).cpu().numpy()
        assert (U == np.eye(n, dtype=np.float32)).all()


def test_inplace_and_determinism(g):
    n, m = 256, 1000
    th, X, dY, _ = _inputs(n, m, seed=1)
    tt, Xt, dYt = _cuda(th), _cuda(X), _cuda(dY)
    Y = g.apply(tt, Xt)
    Xi = Xt.clone()
    g.apply(tt, Xi, out=Xi)
    assert torch.equal(Xi, Y)
    d1, x1 = g.backward(tt, Y, dYt)
    d2, x2 = g.backward(tt, Y, dYt)
    assert torch.equal(d1, d2) and torch.equal(x1, x2)
    dYi = dYt.clone()
    d3, _ = g.backward(tt, Y, dYi, dX=dYi)
    assert torch.equal(d3, d1) and torch.equal(dYi, x1)


def test_autograd_function(g):
    n, m = 128, 64
    th, X, dY, _ = _inputs(n, m, seed=4)
    tt = _cuda(th).requires_grad_(True)
    Xt = _cuda(X).requires_grad_(True)
    Y = g.givens_apply(tt, Xt)
    Y.backward(_cuda(dY))
    dto, dXo = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64))
    assert rel(tt.grad.cpu().numpy(), dto) <= TOL_DTH
    assert rel(Xt.grad.cpu().numpy(), dXo) <= TOL_Y


def test_strided_leading_dimension(g):
    n, m = 64, 100
    th, X, dY, _ = _inputs(n, m, seed=6)
    big = torch.zeros(n, 160, device="cuda")
    big[:, 7:7 + m] = _cuda(X)
    Xv = big[:, 7:7 + m]
    Y = g.apply(_cuda(th), Xv).cpu().numpy()
    assert rel(Y, oracle.apply(n, th, X.astype(np.float64))) <= TOL_Y


@pytest.mark.parametrize("n", [8, 48, 64, 255, 256, 1024, 1120, 2000, 2047, 4096])
def test_fast_slab_path_bitwise(g, n):
    """The whole-slab fast load/store path (aligned rows, every column in range) and the general
    path (rows misaligned by one float, per-element checks) run the same arithmetic in the same
    slab decomposition: Y, dX and dtheta must agree bit for bit."""
    m = 4096
    th, X, dY, _ = _inputs(n, m, seed=21)
    tt, Xc, dYc = _cuda(th), _cuda(X), _cuda(dY)
    Y0 = g.apply(tt, Xc)
    dth0, dX0 = g.backward(tt, Y0, dYc)

    def shifted(a):  # same values, base pointer 4 bytes past a 16-byte boundary
        buf = torch.zeros(a.shape[0] * (m + 4) + 4, device="cuda")
        v = buf[1:1 + a.shape[0] * (m + 4)].view(a.shape[0], m + 4)[:, :m]
        v.copy_(a)
        return v
    Xs, dYs = shifted(Xc), shifted(dYc)
    Ys = shifted(torch.zeros_like(Xc))
    g.apply(tt, Xs, out=Ys)
    dXs = shifted(torch.zeros_like(Xc))
    dths, _ = g.backward(tt, Ys, dYs, dX=dXs)
    torch.cuda.synchronize()
    assert torch.equal(Ys, Y0)
    assert torch.equal(dXs, dX0)
    assert torch.equal(dths, dth0)


# ---------------------------------------------------------------- full-size configurations

def _closed_form_block_dtheta(g, n, Y, dY, r_block):
    """dtheta of block b_1 from (Y, dY): (Y dY^T - dY Y^T)_{ij} (Q_e structure)."""
    Y64, dY64 = Y.double(), dY.double()
    C = (Y64 @ dY64.T - dY64 @ Y64.T).cpu().numpy()
    pairs, flat = oracle.schedule(n)
    idx = flat[r_block] >= 0
    return flat[r_block][idx], C[pairs[r_block][idx, 0], pairs[r_block][idx, 1]]


@pytest.mark.parametrize("n,m", [(256, 4096), (1024, 65536)])
def test_full_size_sampled(g, n, m):
    """BASELINE configs C2 / C3 at full size in the bench launch configuration: forward and dX on
    sampled columns vs the oracle (columns are independent), dtheta of block b_1 vs its closed
    form, and shard additivity dtheta(A u B) = dtheta(A) + dtheta(B)."""
    th, X, dY, _ = _inputs(n, m, seed=11)
    tt, Xt, dYt = _cuda(th), _cuda(X), _cuda(dY)
    Y = g.apply(tt, Xt)
    dth, dX = g.backward(tt, Y, dYt)
    cols = np.unique(np.concatenate([np.arange(8), np.random.default_rng(0).integers(0, m, 24), [m - 1]]))
    Yo = oracle.apply(n, th, X[:, cols].astype(np.float64))
    assert rel(Y.cpu().numpy()[:, cols], Yo) <= TOL_Y
    _, dXo = oracle.backward(n, th, X[:, cols].astype(np.float64), dY[:, cols].astype(np.float64))
    assert rel(dX.cpu().numpy()[:, cols], dXo) <= TOL_Y
    f, want = _closed_form_block_dtheta(g, n, Y, dYt, 0)
    assert rel(dth.cpu().numpy()[f], want) <= TOL_DTH
    h = m // 2
    d1, _ = g.backward(tt, Y[:, :h].contiguous(), dYt[:, :h].contiguous(), want_dX=False)
    d2, _ = g.backward(tt, Y[:, h:].contiguous(), dYt[:, h:].contiguous(), want_dX=False)
    assert rel((d1 + d2).cpu().numpy(), dth.cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("n,m", [(4096, 20), (4095, 9), (1535, 11), (2000, 10), (2400, 7)])
def test_multiwarp_ring_parity(g, n, m):
    """C4 sizes: column groups spanning four warps (L = 128 lanes)."""
    th, X, dY, _ = _inputs(n, m, seed=n)
    tt, Xt, dYt = _cuda(th), _cuda(X), _cuda(dY)
    Y = g.apply(tt, Xt)
    dth, dX = g.backward(tt, Y, dYt)
    Yo = oracle.apply(n, th, X.astype(np.float64))
    dto, dXo = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64))
    assert rel(Y.cpu().numpy(), Yo) <= TOL_Y
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y
    Yt = g.apply(tt, Xt, transpose=True).cpu().numpy()
    assert rel(Yt, oracle.apply(n, th, X.astype(np.float64), transpose=True)) <= TOL_Y


def test_c4_ubuild_gradient_full(g):
    """C4 (n=4096): U from all 8.4M angles + the gradient w.r.t. all of them, in the bench
    configuration; U on sampled columns vs the oracle, U^T U = I on a row sample, dtheta of block
    b_1 vs its closed form (Y dY^T - dY Y^T)_{ij} with Y = U, dY = Gamma."""
    n = 4096
    th = synth.theta(n * (n - 1) // 2, seed=4)
    Gm = synth.normal_matrix(n, n, seed=4, tid=synth.TID_GAMMA)
    tt = _cuda(th)
    U = g.build_U(tt, n)
    Gt = _cuda(Gm)
    dth, _ = g.backward(tt, U, Gt, want_dX=False)
    cols = np.array([0, 1, 777, 2048, 4095])
    E = np.zeros((n, cols.size))
    E[cols, np.arange(cols.size)] = 1.0
    Uo_cols = oracle.apply(n, th, E)
    assert np.abs(U.cpu().numpy()[:, cols] - Uo_cols).max() <= 1e-5 * np.sqrt(n)
    Ud = U.double()
    rows = torch.tensor([0, 5, 1000, 4095], device="cuda")
    orth = (Ud[rows] @ Ud.T - torch.eye(n, device="cuda", dtype=torch.float64)[rows]).abs().max().item()
    assert orth <= 1e-4
    f, want = _closed_form_block_dtheta(g, n, U, Gt, 0)
    assert rel(dth.cpu().numpy()[f], want) <= TOL_DTH


def test_c5_odd_masked_subset(g):
    """C5 shape (n=2047, bye vertex, §5 mask m_keep=1024) on a column subset vs the oracle."""
    n, m = 2047, 96
    th, X, dY, mask = _inputs(n, m, seed=5, mask_keep=1024)
    tt, Xt, dYt, mt = _cuda(th), _cuda(X), _cuda(dY), _cuda(mask)
    Y = g.apply(tt, Xt, mask=mt)
    dth, dX = g.backward(tt, Y, dYt, mask=mt)
    Yo = oracle.apply(n, th, X.astype(np.float64), mask=mask)
    dto, dXo = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64), mask=mask)
    assert rel(Y.cpu().numpy(), Yo) <= TOL_Y
    assert rel(dth.cpu().numpy(), dto) <= TOL_DTH
    assert rel(dX.cpu().numpy(), dXo) <= TOL_Y
    assert (dth.cpu().numpy()[mask == 0] == 0).all()


def test_host_pipeline_matches_direct(g):
    """HostPipeline (overlapped H2D) returns the same dtheta as direct calls, batch by batch."""
    n, m = 256, 512
    th = synth.theta(n * (n - 1) // 2, seed=8)
    tt = _cuda(th)
    batches = [(synth.normal_matrix(n, m, seed=s, tid=synth.TID_X), synth.normal_matrix(n, m, seed=s, tid=synth.TID_DY))
               for s in range(3)]
    pipe = g.HostPipeline(tt, n, m)
    pipe.submit(torch.from_numpy(batches[0][0]).pin_memory(), torch.from_numpy(batches[0][1]).pin_memory())
    for k in range(3):
        if k + 1 < 3:
            pipe.submit(torch.from_numpy(batches[k + 1][0]).pin_memory(),
                        torch.from_numpy(batches[k + 1][1]).pin_memory())
        got = pipe.step()
        torch.cuda.synchronize()
        Y = g.apply(tt, _cuda(batches[k][0]))
        want, _ = g.backward(tt, Y, _cuda(batches[k][1]), want_dX=False)
        assert torch.equal(got, want.cpu())


def test_c5_shard_full_launch(g):
    """C5 as one rank of its 8-GPU run, in the bench launch configuration: n = 2047 (odd: the bye),
    32768 columns, the §5 mask m_keep = 1024. Y and dX on sampled columns vs the oracle, pinned angles
    exactly 0, dtheta of the first block vs its closed form (Y dY^T - dY Y^T)_{ij} (pinned entries 0),
    and shard additivity dtheta(A u B) = dtheta(A) + dtheta(B)."""
    n, m = 2047, 32768
    th, X, dY, mask = _inputs(n, m, seed=17, mask_keep=1024)
    tt, Xt, dYt, mt = _cuda(th), _cuda(X), _cuda(dY), _cuda(mask)
    Y = g.apply(tt, Xt, mask=mt)
    dth, dX = g.backward(tt, Y, dYt, mask=mt)
    d = dth.cpu().numpy()
    assert (d[mask == 0] == 0).all()
    cols = np.unique(np.concatenate([np.arange(3), np.random.default_rng(5).integers(0, m, 9), [m - 1]]))
    Xs, dYs = X[:, cols].astype(np.float64), dY[:, cols].astype(np.float64)
    assert rel(Y.cpu().numpy()[:, cols], oracle.apply(n, th, Xs, mask=mask)) <= TOL_Y
    _, dXo = oracle.backward(n, th, Xs, dYs, mask=mask)
    assert rel(dX.cpu().numpy()[:, cols], dXo) <= TOL_Y
    f, want = _closed_form_block_dtheta(g, n, Y, dYt, 0)
    want = np.where(mask[f] == 0, 0.0, want)
    assert rel(d[f], want) <= TOL_DTH
    h = 12288
    d1, _ = g.backward(tt, Y[:, :h].contiguous(), dYt[:, :h].contiguous(), mask=mt, want_dX=False)
    d2, _ = g.backward(tt, Y[:, h:].contiguous(), dYt[:, h:].contiguous(), mask=mt, want_dX=False)
    assert rel((d1 + d2).cpu().numpy(), d) <= 1e-5
