mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev2_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/ev2_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/ev2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/ev2_bench.log
timeout 900 python bench.py --config 3 > gpurun_out/ev2_bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/ev2_bench_c3.log
timeout 900 python bench.py --config 4 --steps 20 --no-cpu-baseline > gpurun_out/ev2_bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/ev2_bench_c4.log
timeout 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/ev2_bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/ev2_bench_c1.log
