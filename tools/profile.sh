#!/bin/bash
# GPU side (under gpurun): the round's profiling evidence, into gpurun_out/$TAG/.
#  1. FP32 peak microbenchmarks (tools/microbench*.cu, built here) with the SM clock sampled by
#     nvidia-smi while they run;
#  2. the ncu launch list of a short bench run (per-kernel share of the C3 step);
#  3. one `ncu --set full` capture (plus the executed-op / local-memory / L2 metrics) of every
#     kernel of one iteration of each hot-path case (tools/prof_cases.py).
# usage: tools/profile.sh TAG [cases...]
TAG=${1:-r2}; shift
CASES=${@:-c3 c2 ub1024 c4 c5 unitary gemm}
OUT=gpurun_out/$TAG
mkdir -p $OUT
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 100 \
    > $OUT/clocks_microbench.csv 2>/dev/null &
SMI=$!
{
  for b in microbench microbench2 microbench5 microbench6; do
    echo "== tools/$b"; for r in 1 2 3; do timeout 120 ./tools/$b || echo "$b failed"; done
  done
} > $OUT/microbench.txt 2>&1
kill $SMI
EXTRA=smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,\
smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,\
smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,\
smsp__sass_inst_executed_op_local_ld.sum,smsp__sass_inst_executed_op_local_st.sum,lts__t_bytes.sum,\
sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.sum,\
sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.sum,\
smsp__sass_inst_executed_op_shared_ld.sum,smsp__sass_inst_executed_op_shared_st.sum
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-ubuild > $OUT/launches.bench.json 2>/dev/null
for c in $CASES; do
  timeout 900 ncu --set full --metrics $EXTRA --clock-control none --import-source on -c 40 -o $OUT/$c \
      python tools/prof_cases.py $c > $OUT/$c.log 2>&1 || echo "ncu $c failed"
  # reports are too large to bring back (gpurun_out <= 64 MiB): export the raw metrics page (and, for
  # the hot kernels, the per-source-line page) here and drop the report
  ncu -i $OUT/$c.ncu-rep --page raw --csv > $OUT/$c.raw.csv 2>/dev/null
  ncu -i $OUT/$c.ncu-rep --page details --csv > $OUT/$c.details.csv 2>/dev/null
  if [ "$c" = "c3" ] || [ "$c" = "c2" ]; then
    ncu -i $OUT/$c.ncu-rep --page source --csv -k regex:k_ring > $OUT/$c.source.csv 2>/dev/null
  fi
  gzip -f $OUT/$c.raw.csv $OUT/$c.details.csv $OUT/$c.source.csv 2>/dev/null
  rm -f $OUT/$c.ncu-rep
done
echo profile-done
