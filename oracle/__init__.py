"""ctypes wrapper for the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs. The product package never imports this module.
See oracle/oracle.c for the paper passages each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC", "-std=c11"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_num_angles.restype = ctypes.c_int64
        L.oracle_num_angles.argtypes = [ctypes.c_int]
        L.oracle_schedule.restype = ctypes.c_int64
        L.oracle_schedule.argtypes = [ctypes.c_int, P, P, P]
        L.oracle_apply_sequence.restype = ctypes.c_int
        L.oracle_apply_sequence.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, P, P, P, P,
                                            ctypes.c_int64, ctypes.c_int]
        L.oracle_apply.restype = ctypes.c_int
        L.oracle_apply.argtypes = [ctypes.c_int, ctypes.c_int64, P, ctypes.c_int, P, P, P, P, ctypes.c_int]
        L.oracle_build_U.restype = ctypes.c_int
        L.oracle_build_U.argtypes = [ctypes.c_int, P, ctypes.c_int, P, P, P]
        L.oracle_backward.restype = ctypes.c_int
        L.oracle_backward.argtypes = [ctypes.c_int, ctypes.c_int64, P, ctypes.c_int, P, P, P, P, P, P]
        L.oracle_alg3.restype = ctypes.c_int
        L.oracle_alg3.argtypes = [ctypes.c_int, P, P, P, P, P, P]
        L.oracle_u_apply.restype = ctypes.c_int
        L.oracle_u_apply.argtypes = [ctypes.c_int, ctypes.c_int64, P, ctypes.c_int, P, P, P, P, P, ctypes.c_int]
        L.oracle_u_backward.restype = ctypes.c_int
        L.oracle_u_backward.argtypes = [ctypes.c_int, ctypes.c_int64, P, ctypes.c_int, P, P, P, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return lib().oracle_num_threads()


def num_angles(n: int) -> int:
    return int(lib().oracle_num_angles(n))


def n_eff(n: int) -> int:
    return n + (n % 2)


def _perm_arg(perm, n):
    if perm is None:
        return None
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    assert perm.shape == (n_eff(n),)
    return perm


def _refl(reflect):
    return -1 if reflect is None else int(reflect)


def schedule(n: int, perm=None):
    """(pairs[R][S][2] int32, flat[R][S] int64) by literal circle-method simulation, starting from
    the sequence perm (a permutation of 0..n_eff-1; None = identity)."""
    ne = n_eff(n)
    R, S = ne - 1, ne // 2
    pairs = np.zeros((R, S, 2), dtype=np.int32)
    flat = np.zeros((R, S), dtype=np.int64)
    N = lib().oracle_schedule(n, _p(_perm_arg(perm, n)), _p(pairs), _p(flat))
    if N < 0:
        raise ValueError(f"bad n={n} or permutation")
    return pairs, flat


def sequence_E(n: int, perm=None) -> np.ndarray:
    """E as an (N, 2) int32 array of the real pairs in flat (block-major) angle order."""
    pairs, flat = schedule(n, perm)
    N = num_angles(n)
    E = np.zeros((N, 2), dtype=np.int32)
    sel = flat >= 0
    E[flat[sel]] = pairs[sel]
    return E


def _mask_arg(mask, N):
    if mask is None:
        return None
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    assert mask.shape == (N,)
    return mask


def apply_sequence(n: int, E: np.ndarray, theta: np.ndarray, A: np.ndarray, mask=None,
                   transpose: bool = False) -> np.ndarray:
    """Algorithm 1 for an arbitrary pair sequence E on a copy of A (n x m fp64)."""
    E = np.ascontiguousarray(E, dtype=np.int32)
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    m = A.shape[1]
    mask = _mask_arg(mask, E.shape[0])
    rc = lib().oracle_apply_sequence(n, m, E.shape[0], _p(E), _p(theta), _p(mask), _p(A), m,
                                     int(transpose))
    assert rc == 0
    return A


def apply(n: int, theta: np.ndarray, X: np.ndarray, mask=None, transpose: bool = False, perm=None,
          reflect=None) -> np.ndarray:
    """Y = U X (or U^T X); perm = circle-method start sequence, reflect = column of U negated."""
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    X = np.ascontiguousarray(X, dtype=np.float64)
    assert X.shape[0] == n and theta.shape == (num_angles(n),)
    Y = np.empty_like(X)
    rc = lib().oracle_apply(n, X.shape[1], _p(_perm_arg(perm, n)), _refl(reflect), _p(theta),
                            _p(_mask_arg(mask, theta.size)), _p(X), _p(Y), int(transpose))
    assert rc == 0
    return Y


def build_U(n: int, theta: np.ndarray, mask=None, perm=None, reflect=None) -> np.ndarray:
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    U = np.empty((n, n), dtype=np.float64)
    rc = lib().oracle_build_U(n, _p(_perm_arg(perm, n)), _refl(reflect), _p(theta),
                              _p(_mask_arg(mask, theta.size)), _p(U))
    assert rc == 0
    return U


def backward(n: int, theta: np.ndarray, X: np.ndarray, dY: np.ndarray, mask=None, want_dX: bool = True,
             perm=None, reflect=None):
    """(dtheta[N] fp64, dX n x m fp64 or None) for Y = U(theta) X with upstream dY."""
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    X = np.ascontiguousarray(X, dtype=np.float64)
    dY = np.ascontiguousarray(dY, dtype=np.float64)
    assert X.shape == dY.shape and X.shape[0] == n
    N = num_angles(n)
    dth = np.zeros(N, dtype=np.float64)
    dX = np.empty_like(X) if want_dX else None
    rc = lib().oracle_backward(n, X.shape[1], _p(_perm_arg(perm, n)), _refl(reflect), _p(theta),
                               _p(_mask_arg(mask, N)), _p(X), _p(dY), _p(dX), _p(dth))
    assert rc == 0
    return dth, dX


def alg3(n: int, theta: np.ndarray, U: np.ndarray, Gamma: np.ndarray, mask=None, perm=None) -> np.ndarray:
    """The paper's Algorithm 3 literally: dL/dtheta given U and Gamma = dL/dU."""
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    U = np.ascontiguousarray(U, dtype=np.float64)
    Gamma = np.ascontiguousarray(Gamma, dtype=np.float64)
    N = num_angles(n)
    dth = np.zeros(N, dtype=np.float64)
    rc = lib().oracle_alg3(n, _p(_perm_arg(perm, n)), _p(theta), _p(_mask_arg(mask, N)), _p(U), _p(Gamma),
                           _p(dth))
    assert rc == 0
    return dth


def mask_from_keep(n: int, m_keep: int, perm=None) -> np.ndarray:
    """Paper §5 restriction: pair (i,j), i<j, is excluded iff i >= m_keep
    (both ends in S-bar = {m_keep..n-1}). Returns uint8 mask in flat angle order."""
    E = sequence_E(n, perm)
    return (E[:, 0] < m_keep).astype(np.uint8)


# ---------------------------------------------------------------- unitary U(n) (Appendix A)

def _c2i(Z):
    """complex128 n x m -> interleaved float64 n x 2m (re, im)."""
    Z = np.ascontiguousarray(Z, dtype=np.complex128)
    return Z.view(np.float64).reshape(Z.shape[0], 2 * Z.shape[1])


def _i2c(A, m):
    return np.ascontiguousarray(A).view(np.complex128).reshape(A.shape[0], m)


def u_apply(n: int, theta, phi, X, mask=None, adjoint: bool = False, perm=None, reflect=None):
    """Y = U(theta, phi) X (Algorithm 4) or U^dagger X; X complex n x m."""
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    phi = np.ascontiguousarray(phi, dtype=np.float32)
    X = np.ascontiguousarray(X, dtype=np.complex128)
    m = X.shape[1]
    Xi = _c2i(X)
    Yi = np.empty_like(Xi)
    rc = lib().oracle_u_apply(n, m, _p(_perm_arg(perm, n)), _refl(reflect), _p(theta), _p(phi),
                              _p(_mask_arg(mask, theta.size)), _p(Xi), _p(Yi), int(adjoint))
    assert rc == 0
    return _i2c(Yi, m)


def u_build_U(n: int, theta, phi, mask=None, perm=None, reflect=None):
    return u_apply(n, theta, phi, np.eye(n, dtype=np.complex128), mask=mask, perm=perm, reflect=reflect)


def u_backward(n: int, theta, phi, X, Gamma, mask=None, want_dX: bool = True, perm=None, reflect=None):
    """(dtheta, dphi, dX) for a real loss of Y = U X with Gamma = dL/dRe(Y) + i dL/dIm(Y)."""
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    phi = np.ascontiguousarray(phi, dtype=np.float32)
    X = np.ascontiguousarray(X, dtype=np.complex128)
    m = X.shape[1]
    N = num_angles(n)
    Xi, Gi = _c2i(X), _c2i(Gamma)
    dXi = np.empty_like(Xi) if want_dX else None
    dth = np.zeros(N)
    dph = np.zeros(N)
    rc = lib().oracle_u_backward(n, m, _p(_perm_arg(perm, n)), _refl(reflect), _p(theta), _p(phi),
                                 _p(_mask_arg(mask, N)), _p(Xi), _p(Gi), _p(dXi), _p(dth), _p(dph))
    assert rc == 0
    return dth, dph, (_i2c(dXi, m) if want_dX else None)
