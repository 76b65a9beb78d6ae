import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth, paper_2106_00003_b200 as g
def rel(a,b): return np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-30)
def cn(n, m, s): return (synth.normal_matrix(n, m, s, 2).astype(np.float64) + 1j * synth.normal_matrix(n, m, s, 3).astype(np.float64))
for n, m in [(8, 5), (16, 7), (48, 9), (256, 33), (1024, 20), (2047, 6)]:
    N=n*(n-1)//2; th=synth.theta(N,seed=1); ph=synth.theta(N,seed=2)
    X=cn(n,m,1); G=cn(n,m,2)
    tt=torch.from_numpy(th).cuda(); pt=torch.from_numpy(ph).cuda()
    Xt=torch.from_numpy(X.astype(np.complex64)).cuda(); Gt=torch.from_numpy(G.astype(np.complex64)).cuda()
    Y=g.u_apply(tt,pt,Xt); Ya=g.u_apply(tt,pt,Xt,adjoint=True)
    dth,dph,dX=g.u_backward(tt,pt,Y,Gt)
    torch.cuda.synchronize()
    Yo=oracle.u_apply(n,th,ph,X); Yao=oracle.u_apply(n,th,ph,X,adjoint=True)
    dto,dpo,dXo=oracle.u_backward(n,th,ph,X,G)
    out=[n,m,"Y",rel(Y.cpu().numpy(),Yo),"Ya",rel(Ya.cpu().numpy(),Yao),"dth",rel(dth.cpu().numpy(),dto),"dph",rel(dph.cpu().numpy(),dpo),"dX",rel(dX.cpu().numpy(),dXo)]
    if n <= 1024:
        U=g.u_build_U(tt,pt,n).cpu().numpy(); Uo=oracle.u_build_U(n,th,ph); out += ["U", np.abs(U-Uo).max()]
    print(*out, flush=True)
