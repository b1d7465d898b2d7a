mkdir -p gpurun_out; rm -f gpurun_out/r4_lloyd3.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r4_lloyd3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r4_lloyd3_pytest.log
for L in 4 8 16 32; do
  echo "== c2 NRR_LLOYD=$L" >> gpurun_out/r4_lloyd3.log
  NRR_LLOYD=$L timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_lloyd3.log 2>&1
done
for c in 1 3; do
  echo "== c$c" >> gpurun_out/r4_lloyd3.log
  timeout 900 python bench.py --no-cpu-baseline --config $c >> gpurun_out/r4_lloyd3.log 2>&1
done
