"""Profiling driver: `steps` hot-path steps (precompute + forward + replay backward) of a config.
Used under ncu (never a bench number)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2106_00003_b200 as g

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--m", type=int, default=65536)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
n, m = a.n, a.m
N = n * (n - 1) // 2
th = torch.from_numpy(synth.theta(N, seed=0)).cuda()
X = torch.from_numpy(synth.normal_matrix(n, m, 0, synth.TID_X)).cuda()
dY = torch.from_numpy(synth.normal_matrix(n, m, 0, synth.TID_DY)).cuda()
ws = g.workspace(g.OP_BACKWARD, n, m)
Y = torch.empty_like(X); dX = torch.empty_like(X); dth = torch.empty(N, device="cuda")
for _ in range(a.steps):
    g.apply(th, X, out=Y, ws=ws)
    g.backward(th, Y, dY, ws=ws, recompute=False, dtheta=dth, dX=dX)
torch.cuda.synchronize()
print("done")
