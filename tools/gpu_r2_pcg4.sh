mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_kernel -c 1 -s 3 -o gpurun_out/r2_pcg4 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_pcg4_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2_pcg4_ncu.log
