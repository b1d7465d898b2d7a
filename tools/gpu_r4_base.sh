mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r4_base_gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r4_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r4_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r4_base_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r4_base_bench.log
timeout 600 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/r4_base_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r4_base_c4.log
