mkdir -p gpurun_out
NRR_PCG=cluster timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 120 --csv --log-file gpurun_out/launches_c3.csv python tools/profile_step.py --config 3 --iters 3 --warmup 2 > gpurun_out/ncu_c3.log 2>&1
