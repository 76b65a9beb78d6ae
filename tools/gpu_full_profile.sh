timeout 900 python bench.py > gpurun_out/bench_${TAG:-r1h}.json 2> gpurun_out/bench_${TAG:-r1h}.err; tail -2 gpurun_out/bench_${TAG:-r1h}.err
timeout 1200 bash tools/profile.sh ${TAG:-r1h}
ls -la gpurun_out
