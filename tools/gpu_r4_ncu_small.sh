mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"assemble_kernel|nn_kernel|terms_kernel|deform_kernel" -c 4 -s 40 -o gpurun_out/r4_small -f python bench.py --steps 3 --warmup 8 --no-cpu-baseline > gpurun_out/r4_small_ncu.log 2>&1
