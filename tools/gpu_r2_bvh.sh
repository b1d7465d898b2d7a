mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "nn or register" > gpurun_out/r2_bvh_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bvh_tests.log
out=gpurun_out/r2_bvh_bench.log; : > $out
for i in 1 2; do
echo "== device BVH" >> $out; timeout 300 python bench.py --no-cpu-baseline >> $out 2>&1
echo "== host BVH" >> $out; NRR_BVH_HOST=1 timeout 300 python bench.py --no-cpu-baseline >> $out 2>&1
done
echo "== c4 device" >> $out; timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> $out 2>&1
echo "== c4 host" >> $out; NRR_BVH_HOST=1 timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> $out 2>&1
NRR_PROF_SETUP=1 timeout 300 python tools/e2e_timing.py > gpurun_out/r2_e2e_timing.log 2>&1
