mkdir -p gpurun_out
out=gpurun_out/nn_sweep.log; : > $out
for h in 0.7 1.0 1.4 2.0; do for cells in 216 512; do
  echo "H=$h CELLS=$cells" >> $out
  NRR_NN_GRID_H=$h NRR_NN_GRID_CELLS=$cells timeout 120 python tools/profile_step.py --iters 10 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().replace('np.float64','')); print(d['nn'])" >> $out 2>&1
done; done
