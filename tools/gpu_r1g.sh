set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "backward or c4 or alg3 or determinism" 2>&1 | tail -3
timeout 300 python tools/f2_probe.py 2>&1 | tail -20
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-ubuild --no-e2e 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('BENCH', b['value'], b['ms_per_step'], b['fwd_ms'], b['bwd_ms'], b['roofline']['frac'], b['clocks'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ring --launch-skip 1 -c 1 -o gpurun_out/bwd_r1g python tools/prof_step.py --steps 1 > gpurun_out/ncu_r1g.log 2>&1
ls -la gpurun_out/
