"""Device ms of the unitary path at n = 1024 on 32768 complex columns (u_apply, u_backward)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2106_00003_b200 as g
n, m = 1024, 32768
N = n * (n - 1) // 2
th = torch.from_numpy(synth.theta(N, seed=0)).cuda(); ph = torch.from_numpy(synth.theta(N, seed=1)).cuda()
X = torch.complex(torch.from_numpy(synth.normal_matrix(n, m, 0, 2)), torch.from_numpy(synth.normal_matrix(n, m, 1, 2))).cuda()
G = torch.complex(torch.from_numpy(synth.normal_matrix(n, m, 0, 3)), torch.from_numpy(synth.normal_matrix(n, m, 1, 3))).cuda()
wsb = g.workspace(g.OP_U_BACKWARD, n, m); wsf = g.workspace(g.OP_U_APPLY, n, m)
Y = g.u_apply(th, ph, X, ws=wsf); g.u_backward(th, ph, Y, G, ws=wsb); torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record(); g.u_apply(th, ph, X, out=Y, ws=wsf); e[1].record(); g.u_backward(th, ph, Y, G, ws=wsb); e[2].record()
torch.cuda.synchronize()
print(f"unitary n={n} m={m}: u_apply {e[0].elapsed_time(e[1]):.2f} ms  u_backward {e[1].elapsed_time(e[2]):.2f} ms")
