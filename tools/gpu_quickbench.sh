# quick: bwd/fwd timings at C3 + a parity subset
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layout.py -x -q -k "backward or apply_parity or layout" 2>&1 | tail -2
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ubuild --no-e2e 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('BENCH', round(b['value']/1e12,4), round(b['ms_per_step'],3), round(b['fwd_ms'],3), round(b['bwd_ms'],3), round(b['roofline']['frac'],4), b['clocks'])"
done
