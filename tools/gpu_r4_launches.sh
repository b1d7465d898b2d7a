mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pcg|nn_kernel|aa_|assemble|terms|deform|energy|pass_decision|sub_invert|coarse" -c 400 --csv --log-file gpurun_out/r4_launches.csv python bench.py --steps 5 --warmup 8 --no-cpu-baseline > gpurun_out/r4_ncu_launches.log 2>&1; echo "rc=$?" >> gpurun_out/r4_ncu_launches.log
