"""Profiling driver (used under ncu, never a bench number): runs `--reps` iterations of one named
hot-path case with the bench's synthetic inputs, so a launch list / --set full capture can be taken
of exactly the kernels that case launches.

cases: c3 (n=1024, m=65536 apply + backward), c2 (n=256, m=4096), ubN (build_U + gradient,
n=N, e.g. ub1024), c4 (build_U + gradient, n=4096), c5 (n=2047, m=32768, mask m_keep=1024), unitary
(n=1024, 32768 complex columns), gemm (the f2 GEMM path at C3)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2106_00003_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("case")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()


def t(x):
    return torch.from_numpy(x).cuda()


def real_case(n, m, mask_keep=None):
    N = n * (n - 1) // 2
    th = t(synth.theta(N, seed=0))
    X, dY = t(synth.normal_matrix(n, m, 0, synth.TID_X)), t(synth.normal_matrix(n, m, 0, synth.TID_DY))
    mask = t(g.mask_from_keep(n, mask_keep)) if mask_keep else None
    ws = g.workspace(g.OP_BACKWARD, n, m)
    Y, dX, dth = torch.empty_like(X), torch.empty_like(X), torch.empty(N, device="cuda")
    for _ in range(a.reps):
        g.apply(th, X, mask=mask, out=Y, ws=ws)
        g.backward(th, Y, dY, mask=mask, ws=ws, recompute=False, dtheta=dth, dX=dX)


def ubuild_case(n):
    N = n * (n - 1) // 2
    th = t(synth.theta(N, seed=0))
    G = t(synth.normal_matrix(n, n, 0, synth.TID_GAMMA))
    ws = g.workspace(g.OP_BACKWARD, n, n)
    U, dth = torch.empty(n, n, device="cuda"), torch.empty(N, device="cuda")
    for _ in range(a.reps):
        g.build_U(th, n, out=U, ws=ws)
        g.backward(th, U, G, ws=ws, recompute=False, dtheta=dth, want_dX=False)


if a.case == "c3":
    real_case(1024, 65536)
elif a.case == "c2":
    real_case(256, 4096)
elif a.case == "c5":
    real_case(2047, 32768, mask_keep=1024)
elif a.case.startswith("ub"):
    ubuild_case(int(a.case[2:]))
elif a.case == "c4":
    ubuild_case(4096)
elif a.case == "unitary":
    n, m = 1024, 32768
    N = n * (n - 1) // 2
    th, ph = t(synth.theta(N, seed=0)), t(synth.theta(N, seed=1))
    X = torch.complex(t(synth.normal_matrix(n, m, 0, synth.TID_X)), t(synth.normal_matrix(n, m, 1, synth.TID_X)))
    G = torch.complex(t(synth.normal_matrix(n, m, 0, synth.TID_DY)), t(synth.normal_matrix(n, m, 1, synth.TID_DY)))
    for _ in range(a.reps):
        Y = g.u_apply(th, ph, X)
        g.u_backward(th, ph, Y, G)
elif a.case == "gemm":
    n, m = 1024, 65536
    N = n * (n - 1) // 2
    th = t(synth.theta(N, seed=0))
    X, dY = t(synth.normal_matrix(n, m, 0, synth.TID_X)), t(synth.normal_matrix(n, m, 0, synth.TID_DY))
    ws = g.gemm_workspace(n, m)
    Y, dX, dth = torch.empty_like(X), torch.empty_like(X), torch.empty(N, device="cuda")
    for _ in range(a.reps):
        g.gemm_apply(th, X, out=Y, ws=ws)
        g.gemm_backward(th, Y, dY, ws=ws, recompute=False, dtheta=dth, dX=dX)
else:
    raise SystemExit(f"unknown case {a.case}")
torch.cuda.synchronize()
print("done", a.case)
