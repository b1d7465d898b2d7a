# host setup breakdown of the one-shot path (config 2) on the GPU box's CPU
mkdir -p gpurun_out
nproc > gpurun_out/setup.log; lscpu | grep -E "Model name|^CPU\(s\)|Thread" >> gpurun_out/setup.log
NRR_PROF_SETUP=1 timeout 300 python tools/setup_timing.py >> gpurun_out/setup.log 2>&1
timeout 300 python tools/e2e_timing.py >> gpurun_out/setup.log 2>&1
