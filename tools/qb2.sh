#!/bin/bash
# quick correctness (incl. multi-warp configs) + bench of both n=1024 ring configurations
python - <<'PY' || exit 1
import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth, paper_2106_00003_b200 as g
def rel(a,b): return np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-30)
for n in [2047, 2048, 4095, 4096]:
    for d in [0,1]:
        got = g.index_trace(n, d).cpu().numpy(); pairs,_ = oracle.schedule(n)
        print("trace", n, d, (got==pairs).all(), flush=True)
for n, m in [(2047,40),(2048,33),(4096,24),(4095,17)]:
    N=n*(n-1)//2; th=synth.theta(N,seed=1); X=synth.normal_matrix(n,m,seed=1,tid=2); dY=synth.normal_matrix(n,m,seed=1,tid=3)
    tt=torch.from_numpy(th).cuda(); Xt=torch.from_numpy(X).cuda(); dYt=torch.from_numpy(dY).cuda()
    Y=g.apply(tt,Xt); dth,dX=g.backward(tt,Y,dYt); torch.cuda.synchronize()
    Yo=oracle.apply(n,th,X.astype(np.float64)); dto,dXo=oracle.backward(n,th,X.astype(np.float64),dY.astype(np.float64))
    print(n,m,"Y",rel(Y.cpu().numpy(),Yo),"dth",rel(dth.cpu().numpy(),dto),"dX",rel(dX.cpu().numpy(),dXo), flush=True)
PY
timeout 300 python tools/quick.py | tail -3
for w in 16 8; do
GIVENS_RING_W=$w python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('W=$w ms/step', d['ms_per_step'], 'fwd', d['fwd_ms'], 'bwd', d['bwd_ms'], 'rot/s %.3e' % d['value'])"
done
python tools/ubuild_times.py 1024 2048 4096
