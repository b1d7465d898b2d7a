# A/B of prebuilt library variants in paper_2206_03410_b200/_ab (lib_<name>.so): $1 = space separated names
mkdir -p gpurun_out
AB=$PWD/paper_2206_03410_b200/_ab
rm -f gpurun_out/r4_ab.log gpurun_out/r4_ab_pytest.log
for v in $1; do
  echo "== pytest $v" >> gpurun_out/r4_ab_pytest.log
  NRR_LIB_PATH=$AB/lib_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "step_parity or register_mm or aa_fixed or bitwise or side_by_side or large_subdomains" >> gpurun_out/r4_ab_pytest.log 2>&1
done
for rep in 1 2; do
  echo "== base rep $rep" >> gpurun_out/r4_ab.log
  timeout 600 python bench.py --no-cpu-baseline --steps 30 ${BENCH_ARGS} >> gpurun_out/r4_ab.log 2>&1
  for v in $1; do
    echo "== $v rep $rep" >> gpurun_out/r4_ab.log
    NRR_LIB_PATH=$AB/lib_$v.so timeout 600 python bench.py --no-cpu-baseline --steps 30 ${BENCH_ARGS} >> gpurun_out/r4_ab.log 2>&1
  done
done
