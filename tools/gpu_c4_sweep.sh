mkdir -p gpurun_out
out=gpurun_out/c4_sweep.log; : > $out
for ag in 8 4 3; do
  echo "AGG_CTAS=$ag" >> $out
  NRR_AGG_CTAS=$ag NRR_PROF_SETUP=1 timeout 300 python tools/profile_step.py --config 4 --iters 6 2>&1 | grep -E "pcg plan|iters" >> $out
done
