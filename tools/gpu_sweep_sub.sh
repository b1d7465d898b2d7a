mkdir -p gpurun_out
out=gpurun_out/sweep_sub.log; : > $out
for s in 16 20 24 32; do
  echo "SUB_ROWS=$s" >> $out
  NRR_SUB_ROWS=$s timeout 120 python tools/profile_step.py --iters 30 >> $out 2>&1
done
