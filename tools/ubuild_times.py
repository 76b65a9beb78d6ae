"""U-build (and U-build + gradient) device time vs n: the paper's Fig. 2 axes."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2106_00003_b200 as g
out = {}
for n in [int(v) for v in (sys.argv[1:] or ["256", "512", "1024", "1120", "2000", "2048", "4096"])]:
    N = n * (n - 1) // 2
    th = torch.from_numpy(synth.theta(N, seed=0)).cuda()
    G = torch.from_numpy(synth.normal_matrix(n, n, 0, synth.TID_GAMMA)).cuda()
    ws = g.workspace(g.OP_BACKWARD, n, n)
    U = torch.empty(n, n, device="cuda"); dth = torch.empty(N, device="cuda")
    def fwd(): g.build_U(th, n, out=U, ws=ws)
    def bwd(): g.backward(th, U, G, ws=ws, recompute=False, dtheta=dth, want_dX=False)
    reps = 3 if n >= 2000 else 10
    for f in (fwd, bwd): f()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf = tb = 0.0
    for _ in range(reps):
        e[0].record(); fwd(); e[1].record(); bwd(); e[2].record(); torch.cuda.synchronize()
        tf += e[0].elapsed_time(e[1]); tb += e[1].elapsed_time(e[2])
    out[n] = {"build_U_ms": tf / reps, "grad_ms": tb / reps}
    print(n, out[n], flush=True)
print(json.dumps(out))
