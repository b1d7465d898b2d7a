mkdir -p gpurun_out
timeout 300 python tools/e2e_timing.py > gpurun_out/e2e_timing.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_a.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-flush > gpurun_out/bench_b.log 2>&1
