# round 2 baseline at HEAD: GPU suite, default bench, reference arm, launch list
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r2_ncu.log
