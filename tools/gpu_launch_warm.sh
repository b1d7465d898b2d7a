# warm-cache launch list of a short config-2 run (kernel durations without cache flush between launches)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file gpurun_out/launches_warm.csv python tools/profile_step.py --iters 5 > gpurun_out/ncu_warm.log 2>&1
python tools/launch_summary.py gpurun_out/launches_warm.csv > gpurun_out/launches_warm_summary.txt 2>&1
