# full ncu capture of one PCG launch (config 2) with source correlation
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_kernel -s 4 -c 1 -o gpurun_out/pcg_full -f python tools/profile_step.py --iters 3 > gpurun_out/ncu_full.log 2>&1
