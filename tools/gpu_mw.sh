timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unitary.py tests/test_gpu_layout.py -x -q -k "multiwarp or c4 or c5 or 2047 or 2048 or 1120 or 1535 or 2000 or 2400 or 4096 or 4095 or restricted or trace" 2>&1 | tail -3
B='python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e'
P='import json,sys; b=json.loads(sys.stdin.read().strip().splitlines()[-1]); u=b.get("ubuild_ms_vs_n",{}); print(round(b["ms_per_step"],3), round(b["fwd_ms"],3), round(b["bwd_ms"],3), {k:(v["build_U_ms"],v["grad_ms"]) for k,v in u.items()})'
echo NEW; timeout 900 $B 2>/dev/null | python -c "$P"
echo OLD2; (cd exp/old2 && timeout 900 $B 2>/dev/null | python -c "$P")
