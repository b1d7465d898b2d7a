mkdir -p gpurun_out
NRR_PROF_SETUP=1 timeout 300 python tools/setup_timing.py > gpurun_out/setup_timing.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
