# config 3 with the round-4 plans (12 cooperative grids of 12 CTAs side by side): 20 consecutive full runs
mkdir -p gpurun_out
out=gpurun_out/r4_c3_stress.log; : > $out
for i in $(seq 1 20); do
  echo "== run $i" >> $out
  timeout 300 python bench.py --config 3 --no-cpu-baseline >> $out 2>&1; echo "rc=$?" >> $out
done
