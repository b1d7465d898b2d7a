# barrier-free PCG exchange (NRR_PCG_POLL): parity subset, then A/B against the grid-barrier build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "step_parity or register_mm or aa_fixed or bitwise or side_by_side or large_subdomains" > gpurun_out/r4_poll_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r4_poll_pytest.log
for rep in 1 2; do
  echo "== poll rep $rep" >> gpurun_out/r4_poll_ab.log
  timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_poll_ab.log 2>&1
  echo "== nopoll rep $rep" >> gpurun_out/r4_poll_ab.log
  NRR_LIB_PATH=$PWD/paper_2206_03410_b200/_ab/lib_nopoll.so timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_poll_ab.log 2>&1
done
echo "== poll c4" >> gpurun_out/r4_poll_ab.log
timeout 600 python bench.py --config 4 --steps 10 --no-cpu-baseline >> gpurun_out/r4_poll_ab.log 2>&1
echo "== nopoll c4" >> gpurun_out/r4_poll_ab.log
NRR_LIB_PATH=$PWD/paper_2206_03410_b200/_ab/lib_nopoll.so timeout 600 python bench.py --config 4 --steps 10 --no-cpu-baseline >> gpurun_out/r4_poll_ab.log 2>&1
