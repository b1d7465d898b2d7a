mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "anderson or aa or register or step" > gpurun_out/r2_aa_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_aa_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pcg|nn_kernel|aa_|assemble|terms|deform|energy|pass_decision|sub_invert|coarse" -c 300 --csv --log-file gpurun_out/r2_aa_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
