# PCG phase probes need a probe build: NRR_BUILD_DEFINES="-DNRR_PCG_PROBES=1" python -m paper_2206_03410_b200.build --force
NRR_PROF=1 timeout 120 python tools/profile_step.py --iters 10 > gpurun_out/prof.log 2>&1
