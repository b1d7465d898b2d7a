mkdir -p gpurun_out; rm -f gpurun_out/r4_refresh.log
for R in 16 64 256; do
  echo "== c2 REFRESH=$R" >> gpurun_out/r4_refresh.log
  NRR_SUB_REFRESH=$R NRR_COARSE_REFRESH=$R timeout 300 python bench.py --no-cpu-baseline --steps 60 >> gpurun_out/r4_refresh.log 2>&1
done
for L in 8 16 32; do
  echo "== c2 LLOYD=$L" >> gpurun_out/r4_refresh.log
  NRR_LLOYD=$L timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_refresh.log 2>&1
done
