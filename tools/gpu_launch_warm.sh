mkdir -p gpurun_out
NRR_SUB_ROWS=${SUB:-16} timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 60 --csv --log-file gpurun_out/launches_warm.csv python tools/profile_step.py --iters 2 --warmup 1 > gpurun_out/ncu_warm.log 2>&1
