"""Device ms of the C3 forward and backward launches (n = 1024, m = 65536), mean of `reps` back to
back after warm-up -- for A/B runs of kernel variants (swap libgivens.so between runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2106_00003_b200 as g

def t(x): return torch.from_numpy(x).cuda()
n, m, reps = 1024, 65536, 10
N = n * (n - 1) // 2
th = t(synth.theta(N, seed=0)); X = t(synth.normal_matrix(n, m, 0, 2)); dY = t(synth.normal_matrix(n, m, 0, 3))
ws = g.workspace(g.OP_BACKWARD, n, m); Y = torch.empty_like(X); dX = torch.empty_like(X); d = torch.empty(N, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
g.apply(th, X, out=Y, ws=ws); g.backward(th, Y, dY, ws=ws, recompute=False, dtheta=d, dX=dX)
tf = tb = 0.0
for _ in range(reps):
    ev[0].record(); g.apply(th, X, out=Y, ws=ws); ev[1].record()
    g.backward(th, Y, dY, ws=ws, recompute=False, dtheta=d, dX=dX); ev[2].record()
    torch.cuda.synchronize()
    tf += ev[0].elapsed_time(ev[1]); tb += ev[1].elapsed_time(ev[2])
print(f"C3 fwd {tf / reps:.3f} ms  bwd {tb / reps:.3f} ms  step {(tf + tb) / reps:.3f} ms")
