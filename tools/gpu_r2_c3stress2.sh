# config 3 with slack SMs: 6 pairs side by side, PCG grids capped at 20 CTAs (120 of 148 SMs)
mkdir -p gpurun_out
out=gpurun_out/r2_c3_stress_slack.log; : > $out
for i in $(seq 1 20); do
  echo "== run $i" >> $out
  timeout 300 python bench.py --config 3 --no-cpu-baseline --pair-ctas 20 >> $out 2>&1; echo "rc=$?" >> $out
done
