mkdir -p gpurun_out; rm -f gpurun_out/r4_c3sweep.log
for S in 6 9 12 18; do
  echo "== c3 streams=$S" >> gpurun_out/r4_c3sweep.log
  timeout 900 python bench.py --no-cpu-baseline --config 3 --pair-streams $S >> gpurun_out/r4_c3sweep.log 2>&1
done
