#!/bin/bash
# quick correctness + short bench (used during development)
timeout 300 python tools/quick.py || exit 1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', d['ms_per_step'], 'fwd', d['fwd_ms'], 'bwd', d['bwd_ms'], 'rot/s %.3e' % d['value'], 'bwd frac', d['roofline']['frac'], d['clocks'])"
