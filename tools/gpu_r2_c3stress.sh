# 20 consecutive full config-3 runs (256 pairs, 6 cooperative PCG grids side by side): hang check
mkdir -p gpurun_out
out=gpurun_out/r2_c3_stress.log; : > $out
for i in $(seq 1 20); do
  echo "== run $i" >> $out
  timeout 300 python bench.py --config 3 --no-cpu-baseline >> $out 2>&1; echo "rc=$?" >> $out
done
