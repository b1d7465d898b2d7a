NRR_PROF=1 timeout 120 python tools/profile_step.py --iters 10 > gpurun_out/prof.log 2>&1
