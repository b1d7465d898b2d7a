mkdir -p gpurun_out
#timeout 1500 python -m pytest tests/test_setup_gpu.py -m gpu -q -s -p no:cacheprovider -x > gpurun_out/r2_setup.log 2>&1; echo "rc=$?" >> gpurun_out/r2_setup.log
NRR_SETUP_PROF=1 python tools/setup_prof.py 1 >> gpurun_out/r2_setup.log 2>&1
NRR_SETUP_PROF=1 python tools/setup_prof.py 2 >> gpurun_out/r2_setup.log 2>&1
NRR_SETUP_PROF=1 python tools/setup_prof.py 4 >> gpurun_out/r2_setup.log 2>&1
