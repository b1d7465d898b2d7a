mkdir -p gpurun_out; rm -f gpurun_out/r4_lloyd4.log
echo "== c4 default" >> gpurun_out/r4_lloyd4.log
timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> gpurun_out/r4_lloyd4.log 2>&1
echo "== c4 NRR_LLOYD_LARGE=1" >> gpurun_out/r4_lloyd4.log
NRR_PROF_SETUP=1 NRR_LLOYD_LARGE=1 timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> gpurun_out/r4_lloyd4.log 2> gpurun_out/r4_lloyd4_plan.txt
echo "== c4 NRR_LLOYD_LARGE=1 CAP=3" >> gpurun_out/r4_lloyd4.log
NRR_LLOYD_CAP=3 NRR_LLOYD_LARGE=1 timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> gpurun_out/r4_lloyd4.log 2>&1
NRR_LLOYD_LARGE=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity.py -q -x -p no:cacheprovider -k "large_subdomains or config4 or cfg4 or million" > gpurun_out/r4_lloyd4_pytest.log 2>&1
