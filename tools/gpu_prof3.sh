mkdir -p gpurun_out
NRR_PROF=1 timeout 120 python tools/profile_step.py --iters 10 > gpurun_out/prof.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
