mkdir -p gpurun_out
: > gpurun_out/prof.log
for s in 16; do echo "SUB_ROWS=$s" >> gpurun_out/prof.log; NRR_PROF=1 NRR_SUB_ROWS=$s timeout 120 python tools/profile_step.py --iters 10 >> gpurun_out/prof.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
