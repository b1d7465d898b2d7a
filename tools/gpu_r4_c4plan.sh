mkdir -p gpurun_out
NRR_PROF_SETUP=1 timeout 600 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/r4_c4.log 2> gpurun_out/r4_c4_plan.txt
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/r4_c2.log 2>&1
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/r4_c3.log 2>&1
