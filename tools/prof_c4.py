"""Profiling driver for C4: U-build (n=4096) + gradient, one call each (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2106_00003_b200 as g
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
N = n * (n - 1) // 2
th = torch.from_numpy(synth.theta(N, seed=0)).cuda()
G = torch.from_numpy(synth.normal_matrix(n, n, 0, synth.TID_GAMMA)).cuda()
ws = g.workspace(g.OP_BACKWARD, n, n)
U = g.build_U(th, n, ws=ws)
d, _ = g.backward(th, U, G, ws=ws, recompute=False, want_dX=False)
torch.cuda.synchronize()
print("done")
