"""Device times of the latency-regime configurations (C2 and the U-build at n <= 1024), for A/B runs of
launch configurations (e.g. GIVENS_RING_W=8): mean of 50 back-to-back calls behind a GPU spin."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2106_00003_b200 as g

def t(x): return torch.from_numpy(x).cuda()

def timed(fn, reps=50):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us

n, m = 256, 4096
N = n * (n - 1) // 2
th = t(synth.theta(N, seed=0)); X = t(synth.normal_matrix(n, m, 0, 2)); dY = t(synth.normal_matrix(n, m, 0, 3))
ws = g.workspace(g.OP_BACKWARD, n, m); Y = torch.empty_like(X); dX = torch.empty_like(X); d = torch.empty(N, device="cuda")
f = timed(lambda: g.apply(th, X, out=Y, ws=ws))
b = timed(lambda: g.backward(th, Y, dY, ws=ws, recompute=False, dtheta=d, dX=dX))
print(f"C2 fwd {f:.1f} us  bwd {b:.1f} us  total {f + b:.1f} us")
for n in (256, 512, 1024):
    N = n * (n - 1) // 2
    th = t(synth.theta(N, seed=0)); G = t(synth.normal_matrix(n, n, 0, 4))
    ws = g.workspace(g.OP_BACKWARD, n, n); U = torch.empty(n, n, device="cuda"); d = torch.empty(N, device="cuda")
    f = timed(lambda: g.build_U(th, n, out=U, ws=ws))
    b = timed(lambda: g.backward(th, U, G, ws=ws, recompute=False, dtheta=d, want_dX=False))
    print(f"U-build n={n}: build {f:.1f} us  grad {b:.1f} us")
