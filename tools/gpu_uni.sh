timeout 1200 python -m pytest tests/test_gpu_unitary.py tests/test_gpu_layout.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; b=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(b["unitary"])'
