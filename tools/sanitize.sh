#!/bin/bash
# GPU side: compute-sanitizer memcheck / racecheck / synccheck / initcheck over every kernel family at
# small sizes (tools/sanitize_small.py N runs the sizes with n <= N), logs into gpurun_out/$TAG/.
TAG=${1:-san}; MAXN=${2:-256}
OUT=gpurun_out/$TAG; mkdir -p $OUT
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_small.py $MAXN > $OUT/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $OUT/$tool.log | tail -2 | tr '\n' ' ')"
done
