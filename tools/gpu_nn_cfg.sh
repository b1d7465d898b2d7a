mkdir -p gpurun_out; : > gpurun_out/nn_cfg.log
for c in 1 4; do for g in 1 0; do echo "config $c grid $g" >> gpurun_out/nn_cfg.log; NRR_NN_GRID=$g timeout 300 python tools/profile_step.py --config $c --iters 5 2>&1 | tail -2 >> gpurun_out/nn_cfg.log; done; done
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
