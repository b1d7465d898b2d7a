# config 3 after the PCG parity double-buffering: GPU PCG parity tests, then 20 consecutive full runs
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity.py tests/test_sharding.py -m gpu -q -p no:cacheprovider > gpurun_out/r2_fix_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fix_tests.log
out=gpurun_out/r2_c3_stress_fixed.log; : > $out
for i in $(seq 1 20); do
  echo "== run $i" >> $out
  timeout 300 python bench.py --config 3 --no-cpu-baseline >> $out 2>&1; echo "rc=$?" >> $out
done
