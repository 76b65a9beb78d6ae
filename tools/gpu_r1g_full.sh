timeout 900 python bench.py > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err; tail -2 gpurun_out/bench_r1g.err
timeout 1200 bash tools/profile.sh r1g
ls -la gpurun_out
