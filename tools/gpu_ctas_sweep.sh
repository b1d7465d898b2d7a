mkdir -p gpurun_out; : > gpurun_out/ctas.log
for g in 148 132 120 96 74; do echo "CTAS=$g $(timeout 120 python tools/profile_step.py --iters 30 --max-ctas $g 2>&1 | grep iters)" >> gpurun_out/ctas.log; done
