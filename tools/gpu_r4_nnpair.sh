mkdir -p gpurun_out; rm -f gpurun_out/r4_nnpair.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity.py tests/test_landmarks.py -q -x -p no:cacheprovider > gpurun_out/r4_nnpair_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r4_nnpair_pytest.log
for P in 1 0 1 0; do
  echo "== c2 NRR_NN_PAIR=$P" >> gpurun_out/r4_nnpair.log
  NRR_NN_PAIR=$P timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_nnpair.log 2>&1
done
for c in 4 1; do for P in 1 0; do
  echo "== c$c NRR_NN_PAIR=$P" >> gpurun_out/r4_nnpair.log
  NRR_NN_PAIR=$P timeout 600 python bench.py --no-cpu-baseline --config $c --steps 10 >> gpurun_out/r4_nnpair.log 2>&1
done; done
