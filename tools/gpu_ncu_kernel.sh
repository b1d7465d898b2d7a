# full ncu capture of one launch of kernel $1 (config 2 profile run) with source correlation
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s ${2:-4} -c 1 -o gpurun_out/$1_full -f python tools/profile_step.py --iters 3 > gpurun_out/ncu_$1.log 2>&1
