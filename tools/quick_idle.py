import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth, paper_2106_00003_b200 as g
def rel(a,b): return np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-30)
ns = [48, 96, 160, 768, 1120, 1535, 2000, 2400]
for n in ns:
    for d in [0, 1]:
        got = g.index_trace(n, d).cpu().numpy(); pairs,_ = oracle.schedule(n)
        print("trace", n, d, (got==pairs).all(), flush=True)
for n in ns:
    m = 37 if n < 1000 else 9
    N=n*(n-1)//2; th=synth.theta(N,seed=2); X=synth.normal_matrix(n,m,seed=2,tid=2); dY=synth.normal_matrix(n,m,seed=2,tid=3)
    tt=torch.from_numpy(th).cuda(); Xt=torch.from_numpy(X).cuda(); dYt=torch.from_numpy(dY).cuda()
    Y=g.apply(tt,Xt); dth,dX=g.backward(tt,Y,dYt); Yt=g.apply(tt,Xt,transpose=True); torch.cuda.synchronize()
    Yo=oracle.apply(n,th,X.astype(np.float64)); dto,dXo=oracle.backward(n,th,X.astype(np.float64),dY.astype(np.float64))
    Yto=oracle.apply(n,th,X.astype(np.float64),transpose=True)
    print(n,m,"Y",rel(Y.cpu().numpy(),Yo),"Yt",rel(Yt.cpu().numpy(),Yto),"dth",rel(dth.cpu().numpy(),dto),"dX",rel(dX.cpu().numpy(),dXo), flush=True)
