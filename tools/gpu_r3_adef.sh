# A-DEF2 first light: parity subset, then config 2 / 4 benches (A-DEF2 vs additive)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "step_parity or register_mm or aa_fixed or bitwise or side_by_side" > gpurun_out/r3_adef_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3_adef_pytest.log
NRR_PROF_SETUP=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r3_adef_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r3_adef_bench.log
NRR_COARSE_MODE=additive timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r3_add_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r3_add_bench.log
NRR_PROF_SETUP=1 timeout 600 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/r3_adef_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r3_adef_c4.log
