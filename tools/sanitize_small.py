"""Small apply/backward/build_U runs over every kernel family, for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_2106_00003_b200 as g
sizes = [(8, 40), (12, 7), (64, 33), (256, 50), (1024, 20), (2047, 9), (4096, 5)]
if len(sys.argv) > 1:
    sizes = [s for s in sizes if s[0] <= int(sys.argv[1])]
for n, m in sizes:
    N = n * (n - 1) // 2
    th = torch.from_numpy(synth.theta(N, seed=1)).cuda()
    X = torch.from_numpy(synth.normal_matrix(n, m, 1, 2)).cuda()
    dY = torch.from_numpy(synth.normal_matrix(n, m, 1, 3)).cuda()
    mask = torch.from_numpy(synth.random_mask(N, 0.7, seed=1)).cuda()
    Y = g.apply(th, X, mask=mask)
    Yt = g.apply(th, X, transpose=True)
    d, dX = g.backward(th, Y, dY, mask=mask)
    U = g.build_U(th, n) if n <= 1024 else None
    g.index_trace(n, 0); g.index_trace(n, 1)
    torch.cuda.synchronize()
    print("ok", n, m, flush=True)
