"""GEMM path: parity vs the oracle at small sizes, then C3 timings next to the ring."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2106_00003_b200 as g

def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for n, m in [(8, 16), (33, 40), (256, 300), (1024, 500)]:
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=1); X = synth.normal_matrix(n, m, 1, synth.TID_X); dY = synth.normal_matrix(n, m, 1, synth.TID_DY)
    tt, Xt, dYt = (torch.from_numpy(a).cuda() for a in (th, X, dY))
    ws = g.gemm_workspace(n, m)
    Y = g.gemm_apply(tt, Xt, ws=ws)
    Yt = g.gemm_apply(tt, Xt, transpose=True)
    dth, dX = g.gemm_backward(tt, Y, dYt, ws=ws, recompute=False)
    Yo = oracle.apply(n, th, X.astype(np.float64)); Yto = oracle.apply(n, th, X.astype(np.float64), transpose=True)
    dto, dXo = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64))
    print(n, m, "Y", rel(Y.cpu().numpy(), Yo), "Yt", rel(Yt.cpu().numpy(), Yto), "dth", rel(dth.cpu().numpy(), dto),
          "dX", rel(dX.cpu().numpy(), dXo), flush=True)
n, m = 1024, 65536
N = n * (n - 1) // 2
th = torch.from_numpy(synth.theta(N, seed=0)).cuda()
X = torch.from_numpy(synth.normal_matrix(n, m, 0, synth.TID_X)).cuda()
dY = torch.from_numpy(synth.normal_matrix(n, m, 0, synth.TID_DY)).cuda()
ws = g.gemm_workspace(n, m); Y = torch.empty_like(X); dX = torch.empty_like(X); dth = torch.empty(N, device="cuda")
flush = torch.empty(64 << 20, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for it in range(6):
    flush.fill_(1.0)
    ev[0].record(); g.gemm_apply(th, X, out=Y, ws=ws); ev[1].record()
    g.gemm_backward(th, Y, dY, ws=ws, recompute=False, dtheta=dth, dX=dX); ev[2].record()
    torch.cuda.synchronize()
    print("C3 gemm path fwd %.3f ms bwd %.3f ms total %.3f" % (ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[0].elapsed_time(ev[2])), flush=True)
Yr = g.apply(th, X)
print("C3 Y rel vs ring", float((Y - Yr).norm() / Yr.norm()))
dthr, dXr = g.backward(th, Yr, dY)
print("C3 dth rel vs ring", float((dth - dthr).norm() / dthr.norm()), "dX", float((dX - dXr).norm() / dXr.norm()))
