mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_headline_parity.py > gpurun_out/r2_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest_gpu.log
for A in 8 4; do echo "== NRR_AGG_CTAS=$A" >> gpurun_out/r2_agg.log; NRR_AGG_CTAS=$A timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r2_agg.log 2>&1; done
