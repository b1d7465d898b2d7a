mkdir -p gpurun_out
timeout 120 python tools/profile_step.py --iters 10 > gpurun_out/prof.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "nn or step" > gpurun_out/pytest_gpu.log 2>&1
