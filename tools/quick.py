import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth, paper_2106_00003_b200 as g
def rel(a,b): return np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-30)
for n in [8, 6, 256, 1024, 2047]:
    for direction in [0,1]:
        got = g.index_trace(n, direction).cpu().numpy(); pairs,_ = oracle.schedule(n)
        print("trace", n, direction, (got==pairs).all(), flush=True)
for n, m in [(8,16),(6,5),(7,33),(256,100),(1024,300),(2047,64),(100,40)]:
    N=n*(n-1)//2; th=synth.theta(N,seed=1); X=synth.normal_matrix(n,m,seed=1,tid=2); dY=synth.normal_matrix(n,m,seed=1,tid=3)
    tt=torch.from_numpy(th).cuda(); Xt=torch.from_numpy(X).cuda(); dYt=torch.from_numpy(dY).cuda()
    Y=g.apply(tt,Xt); torch.cuda.synchronize()
    Yo=oracle.apply(n,th,X.astype(np.float64))
    dth,dX=g.backward(tt,Y,dYt); torch.cuda.synchronize()
    dto,dXo=oracle.backward(n,th,X.astype(np.float64),dY.astype(np.float64))
    print(n,m,"Y",rel(Y.cpu().numpy(),Yo),"dth",rel(dth.cpu().numpy(),dto),"dX",rel(dX.cpu().numpy(),dXo), flush=True)
