# round 2: headline-size parity tests (teacher-forced), then the full GPU suite and the default bench
mkdir -p gpurun_out
nproc > gpurun_out/r2_host.txt; lscpu | head -20 >> gpurun_out/r2_host.txt
timeout 2400 python -m pytest tests/test_headline_parity.py -m gpu -q -s -p no:cacheprovider > gpurun_out/r2_headline.log 2>&1; echo "rc=$?" >> gpurun_out/r2_headline.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_headline_parity.py > gpurun_out/r2_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
