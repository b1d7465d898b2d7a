mkdir -p gpurun_out
AB=$PWD/paper_2206_03410_b200/_ab
NRR_LIB_PATH=$AB/lib_probes.so NRR_PROF=1 timeout 300 python tools/profile_step.py --iters 20 > gpurun_out/r4_poll_probes_c2.log 2>&1
for v in nofence weak; do
  echo "== $v" >> gpurun_out/r4_poll_ab2.log
  NRR_LIB_PATH=$AB/lib_$v.so timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_poll_ab2.log 2>&1
done
