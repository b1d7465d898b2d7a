# preconditioner refresh-interval sweep on config 2 (device ms per pass, PCG iterations per pass)
mkdir -p gpurun_out
out=gpurun_out/refresh.log; : > $out
for sr in 1 2 1000; do for cr in 1 2 4 1000; do
  echo "SUB_REFRESH=$sr COARSE_REFRESH=$cr" >> $out
  NRR_SUB_REFRESH=$sr NRR_COARSE_REFRESH=$cr timeout 120 python tools/profile_step.py --iters 30 >> $out 2>&1
done; done
