timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "backward_parity or full_size" 2>&1 | tail -2
B='python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e'
P='import json,sys; b=json.loads(sys.stdin.read().strip().splitlines()[-1]); u=b.get("ubuild_ms_vs_n",{}); print(round(b["ms_per_step"],3), round(b["fwd_ms"],3), round(b["bwd_ms"],3), {k:(v["build_U_ms"],v["grad_ms"]) for k,v in u.items()})'
echo NEW; timeout 900 $B 2>/dev/null | python -c "$P"
echo OLD2; (cd exp/old2 && timeout 900 $B --no-ubuild 2>/dev/null | python -c "$P")
