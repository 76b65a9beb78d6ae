"""PyTorch-facing ops over the C ABI (include/givens.h).

PyTorch supplies device memory, streams and process groups; every step of the method runs in
libgivens.so's sm_100a kernels. These wrappers only check shapes/dtypes and marshal pointers.
"""
from __future__ import annotations

import ctypes
import functools
import itertools

import numpy as np
import torch

from . import _lib
from ._lib import (FLAG_RECOMPUTE, FLAG_REUSE_TABLES, OP_APPLY, OP_BACKWARD, OP_BUILD_U, OP_U_APPLY, OP_U_BACKWARD, OP_U_BUILD_U,
                   check, lib)


def num_angles(n: int) -> int:
    """N = n(n-1)/2."""
    v = int(lib().givens_num_angles(n))
    if v < 0:
        raise ValueError(f"n must be >= 2 (got {n})")
    return v


def n_eff(n: int) -> int:
    return n + (n % 2)


def _np_ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Layout:
    """Layout options of one n: the circle method's start permutation
    (a permutation of 0..n_eff-1, None = identity) and the reflection
    class (column `reflect_col` of U negated, det -1). The permutation is
    checked once on the host here (givens_check_perm) and kept on the device for the kernels."""

    def __init__(self, n: int, perm=None, reflect_col: int | None = None, device=None):
        self.n = int(n)
        self.reflect_col = -1 if reflect_col is None else int(reflect_col)
        if not -1 <= self.reflect_col < self.n:
            raise ValueError(f"reflect_col must be None or in [0, {n}) (got {reflect_col})")
        self.perm_host = None
        self.perm = None
        if perm is not None:
            p = np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
            if p.shape != (n_eff(n),):
                raise ValueError(f"perm must have n_eff = {n_eff(n)} entries (got {p.shape})")
            check(lib().givens_check_perm(n, _np_ptr(p)))
            self.perm_host = p
            self.perm = torch.from_numpy(p).to(device or "cuda")

    def args(self, n: int, device):
        if n != self.n:
            raise ValueError(f"layout is for n={self.n}, not n={n}")
        if self.perm is not None and self.perm.device != torch.device(device):
            self.perm = self.perm.to(device)
        return (None if self.perm is None else ctypes.c_void_p(self.perm.data_ptr())), self.reflect_col


def _lay(layout, n, device):
    return (None, -1) if layout is None else layout.args(n, device)


def schedule(n: int, perm=None):
    """Circle-method schedule (closed form, host side): pairs int32[R][S][2], flat int64[R][S];
    perm = start permutation of 0..n_eff-1 (None = identity)."""
    ne = n_eff(n)
    R, S = ne - 1, ne // 2
    pairs = np.zeros((R, S, 2), dtype=np.int32)
    flat = np.zeros((R, S), dtype=np.int64)
    p = None if perm is None else np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    if p is not None and p.shape != (ne,):
        raise ValueError(f"perm must have n_eff = {ne} entries")
    check(lib().givens_schedule_ex(n, _np_ptr(p), _np_ptr(pairs), _np_ptr(flat)))
    return pairs, flat


def mask_from_dims(n: int, excluded, perm=None) -> np.ndarray:
    """uint8 mask[N]: pair (i,j) pinned iff both i and j are in the excluded dimension set."""
    ex = np.zeros(n, dtype=np.uint8)
    ex[np.asarray(list(excluded), dtype=np.int64)] = 1
    mask = np.zeros(num_angles(n), dtype=np.uint8)
    p = None if perm is None else np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    if p is not None and p.shape != (n_eff(n),):
        raise ValueError(f"perm must have n_eff = {n_eff(n)} entries")
    check(lib().givens_mask_from_dims_ex(n, _np_ptr(p), _np_ptr(ex), _np_ptr(mask)))
    return mask


def mask_from_keep(n: int, m_keep: int, perm=None) -> np.ndarray:
    """Paper §5: exclude every pair inside {m_keep, ..., n-1}."""
    return mask_from_dims(n, range(m_keep, n), perm=perm)


def workspace_bytes(op: int, n: int, m: int) -> int:
    return int(lib().givens_workspace_bytes(op, n, m))


def workspace(op: int, n: int, m: int, device=None) -> torch.Tensor:
    """A workspace for op on `device` (its size depends on that device's SM count)."""
    device = torch.device(device or "cuda")
    with torch.cuda.device(device):
        nb = workspace_bytes(op, n, m)
    if nb == 0:
        raise ValueError(f"bad workspace query op={op} n={n} m={m}")
    ws = torch.empty(nb, dtype=torch.uint8, device=device)
    lib().givens_workspace_reset(ctypes.c_void_p(ws.data_ptr()))  # a reused address carries no stale tables
    return ws


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(dev) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _check_matrix(name, t, n):
    if not (t.is_cuda and t.dtype == torch.float32 and t.dim() == 2 and t.shape[0] == n and t.stride(1) == 1):
        raise ValueError(f"{name} must be a CUDA float32 [n, m] tensor with unit column stride "
                         f"(got {tuple(t.shape)} {t.dtype} {t.device} strides {t.stride()})")


def _same_shape(name, t, ref):
    if tuple(t.shape) != tuple(ref.shape):
        raise ValueError(f"{name} must have shape {tuple(ref.shape)} (got {tuple(t.shape)})")


def _on_device(fn):
    """Run an op with the device of its CUDA tensor arguments current (the library launches on, and
    sizes grids for, the current device), and refuse tensors on different devices."""
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        devs = {t.device for t in itertools.chain(args, kwargs.values()) if isinstance(t, torch.Tensor) and t.is_cuda}
        if len(devs) > 1:
            raise ValueError(f"{fn.__name__}: tensors on different devices {sorted(map(str, devs))}")
        if not devs:
            return fn(*args, **kwargs)
        with torch.cuda.device(devs.pop()):
            return fn(*args, **kwargs)
    return wrapper


def _flags(recompute: bool) -> int:
    return FLAG_RECOMPUTE if recompute else FLAG_REUSE_TABLES


def _check_theta(theta, mask, n):
    N = num_angles(n)
    if not (theta.is_cuda and theta.dtype == torch.float32 and theta.is_contiguous() and theta.numel() == N):
        raise ValueError(f"theta must be a contiguous CUDA float32 tensor of {N} angles")
    if mask is not None and not (mask.is_cuda and mask.dtype == torch.uint8 and mask.is_contiguous()
                                 and mask.numel() == N):
        raise ValueError(f"mask must be a contiguous CUDA uint8 tensor of {N} entries")


@_on_device
def apply(theta: torch.Tensor, X: torch.Tensor, mask: torch.Tensor | None = None, transpose: bool = False,
          out: torch.Tensor | None = None, ws: torch.Tensor | None = None, layout: Layout | None = None) -> torch.Tensor:
    """Y = U(theta) X (or U^T X): Algorithm 2 on the columns of X."""
    n, m = X.shape
    _check_matrix("X", X, n)
    _check_theta(theta, mask, n)
    Y = torch.empty_like(X) if out is None else out
    _check_matrix("out", Y, n)
    _same_shape("out", Y, X)
    if ws is None:
        ws = workspace(OP_APPLY, n, m, X.device)
    check(lib().givens_apply_ex(n, m, _ptr(theta), _ptr(mask), _ptr(X), X.stride(0), _ptr(Y), Y.stride(0),
                                int(bool(transpose)), *_lay(layout, n, X.device), _ptr(ws), ws.numel(),
                                _stream(X.device)))
    return Y


@_on_device
def build_U(theta: torch.Tensor, n: int, mask: torch.Tensor | None = None, out: torch.Tensor | None = None,
            ws: torch.Tensor | None = None, layout: Layout | None = None) -> torch.Tensor:
    """U = U(theta) (Algorithm 2 from U <- I_n)."""
    _check_theta(theta, mask, n)
    U = torch.empty((n, n), dtype=torch.float32, device=theta.device) if out is None else out
    _check_matrix("U", U, n)
    if U.shape[1] != n:
        raise ValueError(f"U must be [{n}, {n}] (got {tuple(U.shape)})")
    if ws is None:
        ws = workspace(OP_BUILD_U, n, n, theta.device)
    check(lib().givens_build_U_ex(n, _ptr(theta), _ptr(mask), _ptr(U), U.stride(0), *_lay(layout, n, theta.device),
                                  _ptr(ws), ws.numel(), _stream(theta.device)))
    return U


@_on_device
def backward(theta: torch.Tensor, Y: torch.Tensor, dY: torch.Tensor, mask: torch.Tensor | None = None,
             want_dX: bool = True, ws: torch.Tensor | None = None, recompute: bool = True,
             dtheta: torch.Tensor | None = None, dX: torch.Tensor | None = None, layout: Layout | None = None):
    """(dtheta, dX) for Y = U(theta) X given Y and dY (replay backward, §4).

    recompute=False reuses the coefficient tables a preceding apply/build_U left in `ws`
    (ws must then be a backward-sized workspace that the forward used with the same theta, mask
    and layout; the library checks this and raises otherwise)."""
    n, m = Y.shape
    _check_matrix("Y", Y, n)
    _check_matrix("dY", dY, n)
    _same_shape("dY", dY, Y)
    _check_theta(theta, mask, n)
    if ws is None:
        ws = workspace(OP_BACKWARD, n, m, Y.device)
        recompute = True
    if dtheta is None:
        dtheta = torch.empty(num_angles(n), dtype=torch.float32, device=Y.device)
    if want_dX and dX is None:
        dX = torch.empty_like(dY)
    if dX is not None:
        _check_matrix("dX", dX, n)
        _same_shape("dX", dX, dY)
    check(lib().givens_backward_ex(n, m, _ptr(theta), _ptr(mask), _ptr(Y), Y.stride(0), _ptr(dY), dY.stride(0),
                                   _ptr(dX), dX.stride(0) if dX is not None else 0, _ptr(dtheta),
                                   _flags(recompute), *_lay(layout, n, Y.device), _ptr(ws),
                                   ws.numel(), _stream(Y.device)))
    return dtheta, dX


# ---------------------------------------------------------------- fast Givens

@_on_device
def fast_apply(theta, X, mask=None, out=None, ws=None):
    """Y = U(theta) X by fast (square-root-free) Givens: 2 FMAs per rotation-column on scaled values
    (n_eff in {8, 16, 32, 64} only)."""
    n, m = X.shape
    _check_matrix("X", X, n)
    _check_theta(theta, mask, n)
    Y = torch.empty_like(X) if out is None else out
    _check_matrix("out", Y, n)
    _same_shape("out", Y, X)
    if ws is None:
        ws = workspace(OP_APPLY, n, m, X.device)
    check(lib().givens_fast_apply(n, m, _ptr(theta), _ptr(mask), _ptr(X), X.stride(0), _ptr(Y), Y.stride(0),
                                  _ptr(ws), ws.numel(), _stream(X.device)))
    return Y


@_on_device
def fast_build_U(theta, n: int, mask=None, out=None, ws=None):
    """U = U(theta) by fast Givens (n_eff in {8, 16, 32, 64} only)."""
    _check_theta(theta, mask, n)
    U = torch.empty((n, n), dtype=torch.float32, device=theta.device) if out is None else out
    _check_matrix("U", U, n)
    if ws is None:
        ws = workspace(OP_BUILD_U, n, n, theta.device)
    check(lib().givens_fast_build_U(n, _ptr(theta), _ptr(mask), _ptr(U), U.stride(0), _ptr(ws), ws.numel(),
                                    _stream(theta.device)))
    return U


# ---------------------------------------------------------------- GEMM path

def gemm_workspace(n: int, m: int, device=None) -> torch.Tensor:
    device = torch.device(device or "cuda")
    with torch.cuda.device(device):
        nb = int(lib().givens_gemm_workspace_bytes(n, m))
    if nb == 0:
        raise ValueError(f"bad GEMM workspace query n={n} m={m}")
    ws = torch.empty(nb, dtype=torch.uint8, device=device)
    lib().givens_workspace_reset(ctypes.c_void_p(ws.data_ptr()))  # the ring tables sit at offset 0
    return ws


@_on_device
def gemm_apply(theta, X, mask=None, transpose: bool = False, out=None, ws=None, layout: Layout | None = None):
    """Y = U(theta) X via U-build (register ring) + a 3xTF32 tensor-core GEMM."""
    n, m = X.shape
    _check_matrix("X", X, n)
    _check_theta(theta, mask, n)
    Y = torch.empty_like(X) if out is None else out
    _check_matrix("out", Y, n)
    _same_shape("out", Y, X)
    if ws is None:
        ws = gemm_workspace(n, m, X.device)
    check(lib().givens_gemm_apply(n, m, _ptr(theta), _ptr(mask), _ptr(X), X.stride(0), _ptr(Y), Y.stride(0),
                                  int(bool(transpose)), *_lay(layout, n, X.device), _ptr(ws), ws.numel(),
                                  _stream(X.device)))
    return Y


@_on_device
def gemm_backward(theta, Y, dY, mask=None, want_dX: bool = True, ws=None, recompute: bool = True,
                  dtheta=None, dX=None, layout: Layout | None = None):
    """(dtheta, dX) via dX = U^T dY, Gamma = (dY Y^T) U (3xTF32 GEMMs) and Alg. 3 on Gamma."""
    n, m = Y.shape
    _check_matrix("Y", Y, n)
    _check_matrix("dY", dY, n)
    _same_shape("dY", dY, Y)
    _check_theta(theta, mask, n)
    if ws is None:
        ws = gemm_workspace(n, m, Y.device)
        recompute = True
    if dtheta is None:
        dtheta = torch.empty(num_angles(n), dtype=torch.float32, device=Y.device)
    if want_dX and dX is None:
        dX = torch.empty_like(dY)
    if dX is not None:
        _check_matrix("dX", dX, n)
        _same_shape("dX", dX, dY)
    check(lib().givens_gemm_backward(n, m, _ptr(theta), _ptr(mask), _ptr(Y), Y.stride(0), _ptr(dY), dY.stride(0),
                                     _ptr(dX), dX.stride(0) if dX is not None else 0, _ptr(dtheta),
                                     _flags(recompute), *_lay(layout, n, Y.device), _ptr(ws),
                                     ws.numel(), _stream(Y.device)))
    return dtheta, dX


def index_trace(n: int, direction: int = 0, device=None) -> torch.Tensor:
    """Row ids the kernels pair per (block, slot), as (min, max): int32 [R][S][2] (device)."""
    ne = n_eff(n)
    out = torch.full((ne - 1, ne // 2, 2), -1, dtype=torch.int32, device=device or "cuda")
    with torch.cuda.device(out.device):
        check(lib().givens_index_trace(n, int(direction), _ptr(out), _stream(out.device)))
    return out


class GivensApply(torch.autograd.Function):
    """Y = U(theta) X with the replay backward. The forward's coefficient tables are kept in a
    backward-sized workspace and reused by the backward (no recompute)."""

    @staticmethod
    def forward(ctx, theta, X, mask=None, layout=None):
        n, m = X.shape
        ws = workspace(OP_BACKWARD, n, m, X.device)
        Y = apply(theta, X, mask=mask, ws=ws, layout=layout)
        ctx.layout = layout
        ctx.save_for_backward(theta, Y, mask if mask is not None else torch.empty(0, device=X.device))
        ctx.ws = ws
        ctx.has_mask = mask is not None
        return Y

    @staticmethod
    def backward(ctx, dY):
        theta, Y, mask = ctx.saved_tensors
        mask = mask if ctx.has_mask else None
        dY = dY.contiguous()
        dtheta, dX = backward(theta, Y, dY, mask=mask, want_dX=ctx.needs_input_grad[1], ws=ctx.ws, recompute=False,
                              layout=ctx.layout)
        return dtheta, dX, None, None


def givens_apply(theta, X, mask=None, layout=None):
    """Differentiable Y = U(theta) X."""
    return GivensApply.apply(theta, X, mask, layout)


def version() -> str:
    return lib().givens_version().decode()


class HostPipeline:
    """Training-style loop over host batches: the host->device copy of batch k+1 (on a copy
    stream, from pinned memory) overlaps the forward + backward of batch k (on the compute stream);
    dtheta of every batch is copied back to pinned host memory.

        pipe = HostPipeline(theta, n, m)
        pipe.submit(X0, dY0)
        for k in range(K):
            if k + 1 < K: pipe.submit(X[k+1], dY[k+1])
            dth_host = pipe.step()          # forward + backward of the oldest submitted batch

    step() returns a pinned host tensor that holds that batch's dtheta when step() returns (it
    waits for the device->host copy; the other submitted batch's copy and compute stay queued). Two
    host buffers alternate, so a result stays valid until the step after next; clone it to keep it.
    step(wait=False) returns (buffer, event) without waiting: the caller synchronises the event.
    """

    def __init__(self, theta, n, m, mask=None, want_dX=False, device=None, allreduce=None):
        dev = device or theta.device
        self.theta, self.mask, self.n, self.m, self.want_dX = theta, mask, n, m, want_dX
        self.allreduce = allreduce
        self.compute = torch.cuda.current_stream(dev)
        self.copy = torch.cuda.Stream(dev)
        self.X = [torch.empty(n, m, device=dev) for _ in range(2)]
        self.dY = [torch.empty(n, m, device=dev) for _ in range(2)]
        self.Y = torch.empty(n, m, device=dev)
        self.dX = torch.empty(n, m, device=dev) if want_dX else None
        self.dth = torch.empty(num_angles(n), device=dev)
        self.dth_host = [torch.empty(num_angles(n), dtype=torch.float32).pin_memory() for _ in range(2)]
        self.d2h_done = [torch.cuda.Event() for _ in range(2)]
        self.ws = workspace(OP_BACKWARD, n, m, dev)
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]
        self.n_sub = 0
        self.n_done = 0

    def submit(self, X_host, dY_host):
        s = self.n_sub % 2
        with torch.cuda.stream(self.copy):
            self.copy.wait_event(self.free[s])       # the compute that last read slot s is done
            self.X[s].copy_(X_host, non_blocking=True)
            self.dY[s].copy_(dY_host, non_blocking=True)
            self.ready[s].record(self.copy)
        self.n_sub += 1

    def step(self, wait: bool = True):
        s = self.n_done % 2
        self.compute.wait_event(self.ready[s])
        apply(self.theta, self.X[s], mask=self.mask, out=self.Y, ws=self.ws)
        backward(self.theta, self.Y, self.dY[s], mask=self.mask, ws=self.ws, recompute=False,
                 dtheta=self.dth, dX=self.dX, want_dX=self.want_dX)
        self.free[s].record(self.compute)
        if self.allreduce is not None:
            self.allreduce(self.dth)
        out = self.dth_host[s]
        out.copy_(self.dth, non_blocking=True)
        self.d2h_done[s].record(self.compute)
        self.n_done += 1
        if not wait:
            return out, self.d2h_done[s]
        self.d2h_done[s].synchronize()
        return out


# ---------------------------------------------------------------- unitary U(n) (Appendix A)

def u_supported(n: int) -> bool:
    return bool(lib().givens_u_supported(n))


def _check_cmatrix(name, t, n):
    if not (t.is_cuda and t.dtype == torch.complex64 and t.dim() == 2 and t.shape[0] == n and t.stride(1) == 1):
        raise ValueError(f"{name} must be a CUDA complex64 [n, m] tensor with unit column stride "
                         f"(got {tuple(t.shape)} {t.dtype} {t.device} strides {t.stride()})")


def _check_phi(phi, n):
    N = num_angles(n)
    if not (phi.is_cuda and phi.dtype == torch.float32 and phi.is_contiguous() and phi.numel() == N):
        raise ValueError(f"phi must be a contiguous CUDA float32 tensor of {N} phase angles")


@_on_device
def u_apply(theta, phi, X, mask=None, adjoint: bool = False, out=None, ws=None, layout: Layout | None = None):
    """Y = U(theta, phi) X or U^dagger X (Algorithm 4), X complex64 [n, m]."""
    n, m = X.shape
    _check_cmatrix("X", X, n)
    _check_theta(theta, mask, n)
    _check_phi(phi, n)
    Y = torch.empty_like(X) if out is None else out
    _check_cmatrix("out", Y, n)
    _same_shape("out", Y, X)
    if ws is None:
        ws = workspace(OP_U_APPLY, n, m, X.device)
    check(lib().givens_u_apply_ex(n, m, _ptr(theta), _ptr(phi), _ptr(mask), _ptr(X), X.stride(0), _ptr(Y),
                                  Y.stride(0), int(bool(adjoint)), *_lay(layout, n, X.device), _ptr(ws), ws.numel(),
                                  _stream(X.device)))
    return Y


@_on_device
def u_build_U(theta, phi, n: int, mask=None, out=None, ws=None, layout: Layout | None = None):
    """U = U(theta, phi) in U(n), complex64 [n, n]."""
    _check_theta(theta, mask, n)
    _check_phi(phi, n)
    U = torch.empty((n, n), dtype=torch.complex64, device=theta.device) if out is None else out
    _check_cmatrix("U", U, n)
    if ws is None:
        ws = workspace(OP_U_BUILD_U, n, n, theta.device)
    check(lib().givens_u_build_U_ex(n, _ptr(theta), _ptr(phi), _ptr(mask), _ptr(U), U.stride(0),
                                    *_lay(layout, n, theta.device), _ptr(ws), ws.numel(), _stream(theta.device)))
    return U


@_on_device
def u_backward(theta, phi, Y, dY, mask=None, want_dX: bool = True, ws=None, recompute: bool = True,
               layout: Layout | None = None):
    """(dtheta, dphi, dX) for a real loss of Y = U X, dY = dL/dRe(Y) + i dL/dIm(Y)."""
    n, m = Y.shape
    _check_cmatrix("Y", Y, n)
    _check_cmatrix("dY", dY, n)
    _same_shape("dY", dY, Y)
    _check_theta(theta, mask, n)
    _check_phi(phi, n)
    if ws is None:
        ws = workspace(OP_U_BACKWARD, n, m, Y.device)
        recompute = True
    N = num_angles(n)
    dtheta = torch.empty(N, dtype=torch.float32, device=Y.device)
    dphi = torch.empty(N, dtype=torch.float32, device=Y.device)
    dX = torch.empty_like(dY) if want_dX else None
    check(lib().givens_u_backward_ex(n, m, _ptr(theta), _ptr(phi), _ptr(mask), _ptr(Y), Y.stride(0), _ptr(dY),
                                     dY.stride(0), _ptr(dX), dX.stride(0) if dX is not None else 0, _ptr(dtheta),
                                     _ptr(dphi), _flags(recompute), *_lay(layout, n, Y.device),
                                     _ptr(ws), ws.numel(), _stream(Y.device)))
    return dtheta, dphi, dX
