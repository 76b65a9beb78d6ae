#!/bin/bash
# A/B timing of library builds on one box: for each .so given (paths relative to the repo root),
# install it as paper_2106_00003_b200/libgivens.so and run the timing scripts; the original library
# is restored at the end. usage: bash tools/ab_libs.sh LIB1 LIB2 ... [-- script1.py script2.py]
cd "$(dirname "$0")/.."
libs=(); scripts=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do libs+=("$1"); shift; done
[ "$1" = "--" ] && shift
scripts=("$@")
[ ${#scripts[@]} -eq 0 ] && scripts=(tools/c3_times.py tools/c2_times.py tools/multiwarp_times.py tools/unitary_times.py)
cp paper_2106_00003_b200/libgivens.so /tmp/libgivens.orig.so
for l in "${libs[@]}"; do
  cp "$l" paper_2106_00003_b200/libgivens.so
  echo "=== $l"
  for s in "${scripts[@]}"; do timeout 600 python "$s" 2>&1 | grep -v Warning; done
done
cp /tmp/libgivens.orig.so paper_2106_00003_b200/libgivens.so
