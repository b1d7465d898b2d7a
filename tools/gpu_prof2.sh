mkdir -p gpurun_out
: > gpurun_out/prof.log
for s in 1 8 16 22; do echo "SUB_ROWS=$s" >> gpurun_out/prof.log; NRR_PROF=1 NRR_SUB_ROWS=$s timeout 120 python tools/profile_step.py --iters 10 >> gpurun_out/prof.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_product_kats.py -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"sub_invert|coarse|pcg" -c 12 --csv --log-file gpurun_out/launches_warm.csv python tools/profile_step.py --iters 2 --warmup 1 > /dev/null 2>&1
