"""GPU edge cases of every entry point: an empty batch (m = 0), the largest n on the generic
kernel (S = n_eff/2 without a ring configuration: n = 4097 odd, n = 8192), and n = 2 / 3 (a
single rotation; the bye with one real pair)."""
import numpy as np
import pytest
import torch

import oracle
from _parity import rel
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_00003_b200 as pkg
    return pkg




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


def _c_backward(g, n, m, tt, Y, dY, dX, dth, flags, ws):
    """givens_backward through the C ABI directly (ws may be None = NULL)."""
    import ctypes
    from paper_2106_00003_b200 import _lib
    P = ctypes.c_void_p
    return _lib.lib().givens_backward(n, m, P(tt.data_ptr()), None, P(Y.data_ptr()), m, P(dY.data_ptr()), m,
                                      P(dX.data_ptr()) if dX is not None else None, m, P(dth.data_ptr()), flags,
                                      None if ws is None else P(ws.data_ptr()), 0 if ws is None else ws.numel(),
                                      P(torch.cuda.current_stream().cuda_stream))


@pytest.mark.parametrize("n,m", [(8, 16), (256, 300), (1024, 100), (100, 33)])
def test_backward_self_contained(g, n, m):
    """givens_backward with flags = 0 on a fresh workspace (no forward ever ran into it) and with
    ws = NULL (stream-ordered allocation inside the call) both give the oracle's dtheta and dX
    (every call is self-contained)."""
    from paper_2106_00003_b200 import _lib
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=n)
    X = synth.normal_matrix(n, m, seed=n, tid=synth.TID_X)
    dY = synth.normal_matrix(n, m, seed=n, tid=synth.TID_DY)
    tt, dYt = torch.from_numpy(th).cuda(), torch.from_numpy(dY).cuda()
    Y = g.apply(tt, torch.from_numpy(X).cuda())
    dto, dXo = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64))
    for ws in [torch.full((g.workspace_bytes(g.OP_BACKWARD, n, m),), 0x7F, dtype=torch.uint8, device="cuda"), None]:
        dth = torch.full((N,), float("nan"), device="cuda")
        dX = torch.empty_like(dYt)
        assert _c_backward(g, n, m, tt, Y, dYt, dX, dth, 0, ws) == 0, _lib.lib().givens_last_error()
        torch.cuda.synchronize()
        assert rel(dth.cpu().numpy(), dto) <= 1e-4
        assert rel(dX.cpu().numpy(), dXo) <= 1e-5


def test_reuse_tables_is_checked(g):
    """GIVENS_FLAG_REUSE_TABLES is refused (GIVENS_EINVAL, nothing enqueued) for a workspace no
    forward filled, for a forward with a different theta / mask, and with ws = NULL; it is accepted
    after a forward with the same inputs and then equals the recomputing backward bitwise."""
    from paper_2106_00003_b200 import _lib
    n, m = 256, 64
    N = n * (n - 1) // 2
    th = torch.from_numpy(synth.theta(N, seed=1)).cuda()
    th2 = th.clone()
    X = torch.from_numpy(synth.normal_matrix(n, m, seed=1, tid=synth.TID_X)).cuda()
    dY = torch.from_numpy(synth.normal_matrix(n, m, seed=1, tid=synth.TID_DY)).cuda()
    ws = g.workspace(g.OP_BACKWARD, n, m)
    dth = torch.empty(N, device="cuda")
    dX = torch.empty_like(dY)
    F = _lib.FLAG_REUSE_TABLES
    assert _c_backward(g, n, m, th, X, dY, dX, dth, F, ws) == _lib.EINVAL
    assert _c_backward(g, n, m, th, X, dY, dX, dth, F, None) == _lib.EINVAL
    Y = g.apply(th2, X, ws=ws)
    assert _c_backward(g, n, m, th, Y, dY, dX, dth, F, ws) == _lib.EINVAL  # tables are th2's
    mask = torch.ones(N, dtype=torch.uint8, device="cuda")
    g.apply(th, X, mask=mask, ws=ws)
    assert _c_backward(g, n, m, th, Y, dY, dX, dth, F, ws) == _lib.EINVAL  # tables carry a mask
    g.apply(th, X, out=Y, ws=ws)
    assert _c_backward(g, n, m, th, Y, dY, dX, dth, F, ws) == 0
    d_ref, x_ref = g.backward(th, Y, dY)
    torch.cuda.synchronize()
    assert torch.equal(dth, d_ref) and torch.equal(dX, x_ref)
    with pytest.raises(g.GivensError):
        g.backward(th2, Y, dY, ws=ws, recompute=False)


def test_python_shape_and_device_checks(g):
    n, m = 16, 8
    th = torch.zeros(n * (n - 1) // 2, device="cuda")
    X = torch.zeros(n, m, device="cuda")
    with pytest.raises(ValueError):
        g.backward(th, X, torch.zeros(n, m + 1, device="cuda"))
    with pytest.raises(ValueError):
        g.apply(th, X, out=torch.zeros(n, m + 3, device="cuda"))
    with pytest.raises(ValueError):
        g.backward(th, X, X.clone(), dX=torch.zeros(n, m - 1, device="cuda"))
    with pytest.raises(ValueError):
        g.gemm_backward(th, X, X.clone(), dX=torch.zeros(n, m + 2, device="cuda"))


def test_host_pipeline_result_is_ready(g):
    """HostPipeline.step() returns dtheta already copied to the host (no caller synchronisation)."""
    n, m = 64, 256
    th = torch.from_numpy(synth.theta(n * (n - 1) // 2, seed=3)).cuda()
    pipe = g.HostPipeline(th, n, m)
    Xh = torch.from_numpy(synth.normal_matrix(n, m, seed=3, tid=synth.TID_X)).pin_memory()
    dYh = torch.from_numpy(synth.normal_matrix(n, m, seed=3, tid=synth.TID_DY)).pin_memory()
    pipe.submit(Xh, dYh)
    got = pipe.step().clone()  # read with no synchronize
    want, _ = g.backward(th, g.apply(th, Xh.cuda()), dYh.cuda(), want_dX=False)
    assert torch.equal(got, want.cpu())
