mkdir -p gpurun_out; rm -f gpurun_out/r4_lloyd.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r4_lloyd_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r4_lloyd_pytest.log
for L in 0 16 8 32; do
  echo "== c2 NRR_LLOYD=$L" >> gpurun_out/r4_lloyd.log
  NRR_LLOYD=$L timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_lloyd.log 2>&1
done
for L in 0 16; do
  echo "== c1 NRR_LLOYD=$L" >> gpurun_out/r4_lloyd.log
  NRR_LLOYD=$L timeout 300 python bench.py --no-cpu-baseline --config 1 >> gpurun_out/r4_lloyd.log 2>&1
  echo "== c3 NRR_LLOYD=$L" >> gpurun_out/r4_lloyd.log
  NRR_LLOYD=$L timeout 900 python bench.py --no-cpu-baseline --config 3 >> gpurun_out/r4_lloyd.log 2>&1
done
NRR_PROF_SETUP=1 timeout 300 python bench.py --no-cpu-baseline --steps 5 2>&1 | grep "pcg plan\|rcb plan" | head -3 > gpurun_out/r4_lloyd_plan.txt
