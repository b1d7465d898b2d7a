# quick A/B: PCG parity subset + config 2 bench (+ optional extra bench args in $1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "step_parity or register_mm or aa_fixed or bitwise or side_by_side or large_subdomains" > gpurun_out/r3_quick_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3_quick_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r3_quick_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r3_quick_bench.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r3_quick_bench2.log 2>&1; echo "rc=$?" >> gpurun_out/r3_quick_bench2.log
if [ -n "$1" ]; then timeout 900 python bench.py --no-cpu-baseline $1 > gpurun_out/r3_quick_extra.log 2>&1; echo "rc=$?" >> gpurun_out/r3_quick_extra.log; fi
