mkdir -p gpurun_out; rm -f gpurun_out/r4_cap2.log
for C in 0 5 10 14; do
  echo "== c2 CAP=$C" >> gpurun_out/r4_cap2.log
  NRR_PROF_SETUP=1 NRR_LLOYD_CAP=$C timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_cap2.log 2> gpurun_out/r4_cap2_plan_$C.txt
done
grep -h "pcg plan" gpurun_out/r4_cap2_plan_*.txt | sort -u > gpurun_out/r4_cap2_plans.txt
