#!/bin/bash
# GPU side (under gpurun): the round-end validation run into gpurun_out/$TAG/ -- the GPU test suite,
# smoke(), the default bench line (and the reference arm), then tools/profile.sh (microbenchmarks,
# ncu launch list, --set full per case). usage: tools/validate.sh TAG
TAG=${1:-r2}
cd "$(dirname "$0")/.."
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q > $OUT/gputest.log 2>&1; echo "gpu tests rc=$?" >> $OUT/gputest.log
tail -2 $OUT/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -3 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
bash tools/profile.sh $TAG > $OUT/profile.log 2>&1; tail -1 $OUT/profile.log
