import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2106_00003_b200 as g
for n in [2048, 2047]:
    N = n * (n - 1) // 2
    th = torch.from_numpy(synth.theta(N, seed=0)).cuda()
    G = torch.from_numpy(synth.normal_matrix(n, n, 0, synth.TID_GAMMA)).cuda()
    ws = g.workspace(g.OP_BACKWARD, n, n); U = torch.empty(n, n, device="cuda"); d = torch.empty(N, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for it in range(4):
        ev[0].record(); g.build_U(th, n, out=U, ws=ws); ev[1].record()
        g.backward(th, U, G, ws=ws, recompute=False, dtheta=d, want_dX=False); ev[2].record(); torch.cuda.synchronize()
    print(os.environ.get("GIVENS_RING_W", "default"), n, "build %.3f grad %.3f" % (ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
