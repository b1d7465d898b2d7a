# A/B of prebuilt library variants (no tests): $1 = names; config 2 and config 4
mkdir -p gpurun_out
AB=$PWD/paper_2206_03410_b200/_ab
rm -f gpurun_out/r4_ab2.log
for rep in 1 2; do
  echo "== base rep $rep" >> gpurun_out/r4_ab2.log
  timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_ab2.log 2>&1
  for v in $1; do
    echo "== $v rep $rep" >> gpurun_out/r4_ab2.log
    NRR_LIB_PATH=$AB/lib_$v.so timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_ab2.log 2>&1
  done
done
echo "== base c4" >> gpurun_out/r4_ab2.log
timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> gpurun_out/r4_ab2.log 2>&1
for v in $1; do
  echo "== $v c4" >> gpurun_out/r4_ab2.log
  NRR_LIB_PATH=$AB/lib_$v.so timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> gpurun_out/r4_ab2.log 2>&1
done
