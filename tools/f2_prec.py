"""Precision probe for M = dY Y^T (n=1024, K=m=65536) in 3xTF32 via cuBLAS: whole-K vs K-chunked."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_2106_00003_b200 as g
n, m = 1024, 65536
Y = torch.from_numpy(synth.normal_matrix(n, m, 21, synth.TID_X)).cuda()
dY = torch.from_numpy(synth.normal_matrix(n, m, 21, synth.TID_DY)).cuda()
ref = dY.double() @ Y.double().T
def split(a):
    h = ((a.view(torch.int32) + 0x1000) & ~0x1fff).view(torch.float32)
    return h, a - h
torch.backends.cuda.matmul.fp32_precision = "tf32"
Yh, Yl = split(Y); Dh, Dl = split(dY)
def m3(a_h, a_l, b_h, b_l):
    return a_h @ b_l.T + a_l @ b_h.T + a_h @ b_h.T
M = m3(Dh, Dl, Yh, Yl)
print("3xTF32 whole K: rel", float((M.double() - ref).norm() / ref.norm()), "max abs", float((M.double() - ref).abs().max()))
for ch in [4096, 1024, 256]:
    Mc = sum(m3(Dh[:, i:i+ch], Dl[:, i:i+ch], Yh[:, i:i+ch], Yl[:, i:i+ch]) for i in range(0, m, ch))
    print(f"3xTF32 chunks of {ch}: rel", float((Mc.double() - ref).norm() / ref.norm()))
torch.backends.cuda.matmul.fp32_precision = "ieee"
Ms = dY @ Y.T
print("SGEMM: rel", float((Ms.double() - ref).norm() / ref.norm()))
# how dtheta error depends on M error: Alg.3 on Gamma = M U with exact-ish M vs 3xTF32 M
th = torch.from_numpy(synth.theta(n * (n - 1) // 2, seed=21)).cuda()
U = g.build_U(th, n)
for name, MM in [("fp64->fp32 M", ref.float()), ("3xTF32 M", M), ("SGEMM M", Ms)]:
    Gam = (MM.double() @ U.double()).float()
    d, _ = g.backward(th, U, Gam, want_dX=False)
    if name.startswith("fp64"):
        d0 = d
    print(name, "dtheta rel vs fp64-M path", float((d - d0).norm() / d0.norm()))
