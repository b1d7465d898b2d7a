# bench lines of the non-headline configs on one GPU
mkdir -p gpurun_out
for c in 1 4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; done
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
