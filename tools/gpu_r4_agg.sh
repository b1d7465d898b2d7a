mkdir -p gpurun_out; rm -f gpurun_out/r4_agg.log
for A in 8 4; do
  echo "== c2 NRR_AGG_CTAS=$A" >> gpurun_out/r4_agg.log
  NRR_AGG_CTAS=$A timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_agg.log 2>&1
done
