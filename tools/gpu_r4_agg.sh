mkdir -p gpurun_out; rm -f gpurun_out/r4_agg.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "step_parity or register_mm or aa_fixed or bitwise or side_by_side or large_subdomains" > gpurun_out/r4_agg_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r4_agg_pytest.log
for A in 8 4; do
  echo "== c2 NRR_AGG_CTAS=$A" >> gpurun_out/r4_agg.log
  NRR_AGG_CTAS=$A timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_agg.log 2>&1
done
echo "== c2 A=4 unaligned" >> gpurun_out/r4_agg.log
NRR_RCB_ALIGN=1 timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_agg.log 2>&1
for A in 8 4; do
  echo "== c1 NRR_AGG_CTAS=$A" >> gpurun_out/r4_agg.log
  NRR_AGG_CTAS=$A timeout 300 python bench.py --no-cpu-baseline --config 1 >> gpurun_out/r4_agg.log 2>&1
  echo "== c3 NRR_AGG_CTAS=$A" >> gpurun_out/r4_agg.log
  NRR_AGG_CTAS=$A timeout 900 python bench.py --no-cpu-baseline --config 3 >> gpurun_out/r4_agg.log 2>&1
done
echo "== c4" >> gpurun_out/r4_agg.log
NRR_PROF_SETUP=1 timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> gpurun_out/r4_agg.log 2> gpurun_out/r4_agg_plan.txt
NRR_PROF_SETUP=1 timeout 300 python bench.py --no-cpu-baseline --steps 3 2>&1 | grep "pcg plan" | head -1 >> gpurun_out/r4_agg_plan.txt
