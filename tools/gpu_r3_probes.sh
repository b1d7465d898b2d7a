# PCG phase probes (probe build on the box; the box copy is discarded after the call)
mkdir -p gpurun_out
NRR_BUILD_DEFINES="-DNRR_PCG_PROBES=1" python -m paper_2206_03410_b200.build --force > gpurun_out/r3_probe_build.log 2>&1
NRR_COARSE_MODE=additive NRR_PROF=1 timeout 300 python tools/profile_step.py --iters 20 > gpurun_out/r3_probes_c2.log 2>&1
NRR_COARSE_MODE=additive NRR_PROF=1 timeout 300 python tools/profile_step.py --config 4 --iters 5 > gpurun_out/r3_probes_c4.log 2>&1
