# quick PCG parameter sweep on config 2 (device ms per MM pass, PCG iterations per pass)
mkdir -p gpurun_out
out=gpurun_out/sweep.log; : > $out
for s in 16 24; do for ag in 8 5 4; do
  echo "SUB_ROWS=$s AGG_CTAS=$ag" >> $out
  NRR_SUB_ROWS=$s NRR_AGG_CTAS=$ag timeout 120 python tools/profile_step.py --iters 10 >> $out 2>&1
done; done
