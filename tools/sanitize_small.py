"""Small apply/backward/build_U runs over every kernel family, for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_2106_00003_b200 as g
sizes = [(8, 40), (12, 7), (64, 33), (256, 50), (256, 64), (1024, 20), (1024, 64), (2047, 9), (2047, 32), (4096, 5), (4096, 16)]
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
# unitary (ring, idle-lane ring, generic), layout options, GEMM path
for n, m in [(7, 5), (48, 9), (64, 6), (256, 12), (100, 4)]:
    if len(sys.argv) > 1 and n > int(sys.argv[1]):
        continue
    N = n * (n - 1) // 2
    th = torch.from_numpy(synth.theta(N, seed=1)).cuda()
    ph = torch.from_numpy(synth.theta(N, seed=2)).cuda()
    X = torch.complex(torch.from_numpy(synth.normal_matrix(n, m, 1, 2)), torch.from_numpy(synth.normal_matrix(n, m, 2, 2))).cuda()
    G = torch.complex(torch.from_numpy(synth.normal_matrix(n, m, 1, 3)), torch.from_numpy(synth.normal_matrix(n, m, 2, 3))).cuda()
    lay = g.Layout(n, perm=np.random.default_rng(n).permutation(n + n % 2), reflect_col=n // 2)
    Y = g.u_apply(th, ph, X, layout=lay)
    g.u_apply(th, ph, X, adjoint=True)
    g.u_backward(th, ph, Y, G, layout=lay)
    g.u_build_U(th, ph, n)
    Xr = X.real.contiguous()
    Yr = g.apply(th, Xr, layout=lay)
    g.backward(th, Yr, G.real.contiguous(), layout=lay)
    ws = g.gemm_workspace(n, m)
    Yg = g.gemm_apply(th, Xr, ws=ws, layout=lay)
    g.gemm_backward(th, Yg, G.real.contiguous(), ws=ws, recompute=False, layout=lay)
    torch.cuda.synchronize()
    print("ok-u/layout/gemm", n, m, flush=True)
