mkdir -p gpurun_out; rm -f gpurun_out/r4_nn_sweep.log
for H in 0.7 0.85 1.0 1.2 1.4; do
  echo "== c2 H=$H" >> gpurun_out/r4_nn_sweep.log
  NRR_NN_GRID_H=$H timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_nn_sweep.log 2>&1
  echo "== c4 H=$H" >> gpurun_out/r4_nn_sweep.log
  NRR_NN_GRID_H=$H timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> gpurun_out/r4_nn_sweep.log 2>&1
done
