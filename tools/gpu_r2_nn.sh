mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2_nn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_nn_tests.log
for T in 1 0; do echo "== NRR_NN_TILED=$T" >> gpurun_out/r2_nn_bench.log; NRR_NN_TILED=$T timeout 300 python bench.py --no-cpu-baseline >> gpurun_out/r2_nn_bench.log 2>&1; NRR_NN_TILED=$T timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> gpurun_out/r2_nn_bench.log 2>&1; done
