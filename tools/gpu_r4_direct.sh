mkdir -p gpurun_out
AB=$PWD/paper_2206_03410_b200/_ab
NRR_LIB_PATH=$AB/lib_direct.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "step_parity or register_mm or aa_fixed or bitwise or side_by_side or large_subdomains or anderson" > gpurun_out/r4_direct_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r4_direct_pytest.log
rm -f gpurun_out/r4_direct_ab.log
for rep in 1 2; do
  echo "== base rep $rep" >> gpurun_out/r4_direct_ab.log
  timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_direct_ab.log 2>&1
  echo "== direct rep $rep" >> gpurun_out/r4_direct_ab.log
  NRR_LIB_PATH=$AB/lib_direct.so timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_direct_ab.log 2>&1
done
for c in 4 1; do
echo "== base c$c" >> gpurun_out/r4_direct_ab.log
timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline >> gpurun_out/r4_direct_ab.log 2>&1
echo "== direct c$c" >> gpurun_out/r4_direct_ab.log
NRR_LIB_PATH=$AB/lib_direct.so timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline >> gpurun_out/r4_direct_ab.log 2>&1
done
