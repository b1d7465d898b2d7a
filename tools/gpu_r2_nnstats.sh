mkdir -p gpurun_out
for C in 2 4; do NRR_NN_STATS=1 timeout 600 python bench.py --no-cpu-baseline --config $C --steps 5 --warmup 3 > /dev/null 2> gpurun_out/r2_nnstats_$C.log; done
