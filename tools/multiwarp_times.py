"""Device times of the multi-warp column configurations (n = 2047 / 2048 / 4096): the C5 shard
(n = 2047, 32768 columns, mask m_keep = 1024), the U-build and its gradient at n = 2048 and 4096
(C4); mean of `reps` calls back to back after a warm-up."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2106_00003_b200 as g

def t(x): return torch.from_numpy(x).cuda()

def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

n, m = 2047, 32768
N = n * (n - 1) // 2
th = t(synth.theta(N, seed=0)); mask = t(g.mask_from_keep(n, 1024))
X = t(synth.normal_matrix(n, m, 0, 2)); dY = t(synth.normal_matrix(n, m, 0, 3))
ws = g.workspace(g.OP_BACKWARD, n, m); Y = torch.empty_like(X); dX = torch.empty_like(X); d = torch.empty(N, device="cuda")
f = timed(lambda: g.apply(th, X, mask=mask, out=Y, ws=ws))
b = timed(lambda: g.backward(th, Y, dY, mask=mask, ws=ws, recompute=False, dtheta=d, dX=dX))
print(f"C5 shard fwd {f:.3f} ms  bwd {b:.3f} ms")
for n in (2048, 4096):
    N = n * (n - 1) // 2
    th = t(synth.theta(N, seed=0)); G = t(synth.normal_matrix(n, n, 0, 4))
    ws = g.workspace(g.OP_BACKWARD, n, n); U = torch.empty(n, n, device="cuda"); d = torch.empty(N, device="cuda")
    f = timed(lambda: g.build_U(th, n, out=U, ws=ws))
    b = timed(lambda: g.backward(th, U, G, ws=ws, recompute=False, dtheta=d, want_dX=False))
    print(f"U-build n={n}: build {f:.3f} ms  grad {b:.3f} ms")
