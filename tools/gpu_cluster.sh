mkdir -p gpurun_out
NRR_PCG=cluster timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -p no:cacheprovider > gpurun_out/pytest_cluster.log 2>&1
NRR_PCG=cluster timeout 300 python tools/profile_step.py --config 3 --iters 10 > gpurun_out/prof_c3_cluster.log 2>&1
timeout 300 python tools/profile_step.py --config 3 --iters 10 > gpurun_out/prof_c3_grid.log 2>&1
