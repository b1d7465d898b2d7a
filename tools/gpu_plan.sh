mkdir -p gpurun_out
for c in 2 4; do NRR_PROF_SETUP=1 NRR_PROF=1 timeout 300 python tools/profile_step.py --config $c --iters 5 > gpurun_out/plan_c$c.log 2>&1; done
