mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config 3 --pairs 16 > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --config 1 --steps 20 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1
