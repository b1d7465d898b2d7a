mkdir -p gpurun_out
: > gpurun_out/sweep.log
for w in 0 2 6 12 30; do
  echo "RCB_W=$w" >> gpurun_out/sweep.log
  NRR_RCB_W=$w timeout 120 python tools/profile_step.py --iters 10 2>&1 | grep "iters 10" >> gpurun_out/sweep.log
done
