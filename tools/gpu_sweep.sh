mkdir -p gpurun_out
: > gpurun_out/sweep.log
for agg in 4 8 16; do for sub in 12 16 22; do
  echo "AGG=$agg SUB=$sub" >> gpurun_out/sweep.log
  NRR_AGG_CTAS=$agg NRR_SUB_ROWS=$sub timeout 120 python tools/profile_step.py --iters 10 2>&1 | grep "iters 10" >> gpurun_out/sweep.log
done; done
