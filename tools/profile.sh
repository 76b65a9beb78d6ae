#!/bin/bash
# GPU side: launch list of a short bench run + one --set full capture of the ring kernels.
# usage (under gpurun): tools/profile.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-ubuild > gpurun_out/launches_${TAG}.bench.json 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:k_ring -c 2 -o gpurun_out/ring_${TAG} \
    python tools/prof_step.py --steps 1 > /dev/null 2>&1
echo profile-done
