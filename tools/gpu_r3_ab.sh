# A/B of compile-time variants: $1 = space-separated list of NRR_BUILD_DEFINES sets joined by ','
# e.g. bash tools/gpu_r3_ab.sh "-DNRR_AB_ZZ=1,-DNRR_AB_SYNC6=1,-DNRR_AB_ZZ=1 -DNRR_AB_SYNC6=1"
mkdir -p gpurun_out /tmp/ab
IFS=',' read -ra VARS <<< "$1"
i=0
for v in "" "${VARS[@]}"; do
  touch paper_2206_03410_b200/csrc/pcg.cu
  NRR_BUILD_DEFINES="$v" python -m paper_2206_03410_b200.build > gpurun_out/r3_ab_build_$i.log 2>&1
  cp paper_2206_03410_b200/libnrr_b200.so /tmp/ab/lib_$i.so
  i=$((i+1))
done
for rep in 1 2; do
  i=0
  for v in "" "${VARS[@]}"; do
    echo "== variant $i [$v] rep $rep" >> gpurun_out/r3_ab.log
    NRR_LIB_PATH=/tmp/ab/lib_$i.so timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} >> gpurun_out/r3_ab.log 2>&1
    i=$((i+1))
  done
done
