# round-4 final evidence at HEAD: tests, bench lines for configs 1-4 (+ CPU baselines), reference arm, launch list,
# full ncu captures of the PCG and the Anderson kernels
mkdir -p gpurun_out
nproc > gpurun_out/ev9_host.txt; lscpu | head -20 >> gpurun_out/ev9_host.txt; nvidia-smi >> gpurun_out/ev9_host.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev9_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/ev9_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/ev9_bench.log 2>&1; echo "rc=$?" >> gpurun_out/ev9_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/ev9_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/ev9_bench_ref.log
timeout 600 python bench.py --config 1 > gpurun_out/ev9_bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/ev9_bench_c1.log
timeout 900 python bench.py --config 3 > gpurun_out/ev9_bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/ev9_bench_c3.log
timeout 1200 python bench.py --config 4 --steps 20 > gpurun_out/ev9_bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/ev9_bench_c4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pcg|nn_kernel|aa_|assemble|terms|deform|energy|pass_decision|sub_invert|coarse" -c 400 --csv --log-file gpurun_out/ev9_launches.csv python bench.py --steps 5 --warmup 8 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_kernel -c 1 -s 3 -o gpurun_out/ev9_pcg -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"aa_push_qr_kernel|aa_solve_kernel" -c 2 -s 12 -o gpurun_out/ev9_aa -f python bench.py --steps 3 --warmup 8 --no-cpu-baseline > /dev/null 2>&1
