# full GPU suite + config 2 bench twice (+ optional extra bench args in $1)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r4_quick_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r4_quick_pytest.log
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/r4_quick_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r4_quick_bench.log
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/r4_quick_bench2.log 2>&1; echo "rc=$?" >> gpurun_out/r4_quick_bench2.log
if [ -n "$1" ]; then timeout 900 python bench.py --no-cpu-baseline $1 > gpurun_out/r4_quick_extra.log 2>&1; echo "rc=$?" >> gpurun_out/r4_quick_extra.log; fi
