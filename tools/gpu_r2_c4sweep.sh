mkdir -p gpurun_out
out=gpurun_out/r2_c4_subrows.log; : > $out
for S in 32 24 16 12; do echo "== NRR_SUB_ROWS=$S" >> $out; NRR_SUB_ROWS=$S timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline >> $out 2>&1; done
