mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r3_base_gpu.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r3_base_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r3_base_bench.log
timeout 600 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/r3_base_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r3_base_c4.log
