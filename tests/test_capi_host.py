"""CPU-only checks of the product library's host side (no compute calls need a GPU):
the C-ABI library loads and exports every symbol include/givens.h declares, the closed-form
host schedule is bit-identical to the oracle's literal circle-method simulation, parameter
errors are reported before anything is enqueued."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def g():
    from paper_2106_00003_b200 import build
    build.build()
    import paper_2106_00003_b200 as pkg
    return pkg


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "givens.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(givens_[a-zA-Z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(g):
    from paper_2106_00003_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    decl = _declared_functions()
    assert len(decl) >= 10
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(_lib.EXPORTS)


def test_library_is_sm100a(g):
    from paper_2106_00003_b200 import _lib
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n", list(range(2, 80)) + [127, 128, 255, 256, 511, 1023, 1024, 2047, 2048, 4096])
def test_closed_form_schedule_equals_literal(g, n):
    p1, f1 = g.schedule(n)
    p2, f2 = oracle.schedule(n)
    assert (p1 == p2).all() and (f1 == f2).all()


@pytest.mark.parametrize("n,mk", [(8, 4), (9, 3), (64, 17), (2047, 1024), (1024, 1)])
def test_mask_from_keep_matches_oracle(g, n, mk):
    assert (g.mask_from_keep(n, mk) == oracle.mask_from_keep(n, mk)).all()


def test_num_angles_and_workspace(g):
    assert g.num_angles(1024) == 523776
    with pytest.raises(ValueError):
        g.num_angles(1)
    for op in (0, 1, 2):
        assert g.workspace_bytes(op, 1024, 65536) > 4 * 1024 * 1024
    from paper_2106_00003_b200 import _lib
    assert _lib.lib().givens_workspace_bytes(0, 1, 5) == 0
    assert _lib.lib().givens_workspace_bytes(7, 8, 5) == 0


def test_parameter_errors_before_enqueue(g):
    from paper_2106_00003_b200 import _lib
    L = _lib.lib()
    # n < 2
    rc = L.givens_apply(1, 4, None, None, None, 4, None, 4, 0, None, 0, None)
    assert rc == _lib.EINVAL and b"n must be" in L.givens_last_error()
    # NULL workspace is allowed (stream-ordered allocation inside the call), but only after the
    # arguments are validated: NULL data pointers are still refused before anything is allocated
    rc = L.givens_apply(8, 4, None, None, None, 4, None, 4, 0, None, 0, None)
    assert rc == _lib.EINVAL and b"non-NULL" in L.givens_last_error()
    # table reuse needs the forward's workspace
    rc = L.givens_backward(8, 4, ctypes.c_void_p(16), None, ctypes.c_void_p(16), 4, ctypes.c_void_p(16), 4, None, 0,
                           ctypes.c_void_p(16), _lib.FLAG_REUSE_TABLES, None, 0, None)
    assert rc == _lib.EINVAL and b"REUSE" in L.givens_last_error()
    # table reuse of a workspace no forward filled
    rc = L.givens_backward(8, 4, ctypes.c_void_p(16), None, ctypes.c_void_p(16), 4, ctypes.c_void_p(16), 4, None, 0,
                           ctypes.c_void_p(16), _lib.FLAG_REUSE_TABLES, ctypes.c_void_p(1 << 20), 10 ** 9, None)
    assert rc == _lib.EINVAL and b"no forward" in L.givens_last_error()
    # misaligned workspace / too small
    rc = L.givens_apply(8, 4, None, None, None, 4, None, 4, 0, ctypes.c_void_p(256 + 8), 10 ** 9, None)
    assert rc == _lib.EINVAL and b"aligned" in L.givens_last_error()
    rc = L.givens_apply(8, 4, None, None, None, 4, None, 4, 0, ctypes.c_void_p(256), 16, None)
    assert rc == _lib.EINVAL and b"too small" in L.givens_last_error()
    # NULL data pointers
    rc = L.givens_apply(8, 4, None, None, None, 4, None, 4, 0, ctypes.c_void_p(256), 10 ** 9, None)
    assert rc == _lib.EINVAL
    # leading dimension
    rc = L.givens_backward(8, 4, ctypes.c_void_p(16), None, ctypes.c_void_p(16), 2, ctypes.c_void_p(16), 4, None, 0,
                           ctypes.c_void_p(16), 0, ctypes.c_void_p(256), 10 ** 9, None)
    assert rc == _lib.EINVAL and b"leading dimension" in L.givens_last_error()


def test_product_package_does_not_import_oracle():
    """The product path never routes through the oracle (no import, no link, no exec)."""
    pkg = os.path.join(ROOT, "paper_2106_00003_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle/", ""), f


# ---------------------------------------------------------------- layout options (§8(f3))

def _rperm(n, seed):
    return np.random.default_rng(seed).permutation(n + n % 2).astype(np.int32)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 16, 33, 64, 129, 1024, 2047])
@pytest.mark.parametrize("seed", [0, 1])
def test_permuted_schedule_equals_literal(g, n, seed):
    """Host closed form + relabeling == the oracle's literal circle method from the permuted
    start sequence (bit-exact), including where the odd-n bye lands."""
    p = _rperm(n, seed)
    p1, f1 = g.schedule(n, perm=p)
    p2, f2 = oracle.schedule(n, perm=p)
    assert (p1 == p2).all() and (f1 == f2).all()


@pytest.mark.parametrize("n,mk", [(8, 4), (9, 3), (64, 17), (2047, 1024)])
def test_permuted_mask_matches_oracle(g, n, mk):
    p = _rperm(n, n)
    assert (g.mask_from_keep(n, mk, perm=p) == oracle.mask_from_keep(n, mk, perm=p)).all()


def test_layout_validation(g):
    with pytest.raises(g.GivensError):
        g.Layout(6, perm=[0, 1, 2, 3, 4, 4], device="cpu")
    with pytest.raises(g.GivensError):
        g.Layout(5, perm=[0, 1, 2, 3, 6, 5], device="cpu")
    with pytest.raises(ValueError):
        g.Layout(5, perm=[0, 1, 2, 3, 4], device="cpu")  # n_eff = 6 entries needed
    with pytest.raises(ValueError):
        g.Layout(5, reflect_col=5, device="cpu")
    lay = g.Layout(5, perm=[5, 0, 1, 2, 3, 4], reflect_col=4, device="cpu")
    assert lay.reflect_col == 4 and lay.perm_host.tolist() == [5, 0, 1, 2, 3, 4]
    from paper_2106_00003_b200 import _lib
    L = _lib.lib()
    # reflect_col out of range is a parameter error, detected before anything is enqueued
    rc = L.givens_apply_ex(8, 4, None, None, None, 4, None, 4, 0, None, 8, ctypes.c_void_p(256), 10 ** 9, None)
    assert rc == _lib.EINVAL
    assert b"reflect_col" in L.givens_last_error()
