mkdir -p gpurun_out
out=gpurun_out/r2_sweep_nn.log; : > $out
for H in 1.0 1.4 2.0; do for C in 216 1000; do
  echo "== H=$H CELLS=$C" >> $out
  NRR_NN_GRID_H=$H NRR_NN_GRID_CELLS=$C timeout 300 python bench.py --no-cpu-baseline --steps 20 >> $out 2>&1
done; done
for H in 1.0 2.0; do echo "== c4 H=$H" >> $out; NRR_NN_GRID_H=$H timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> $out 2>&1; done
out=gpurun_out/r2_sweep_c3.log; : > $out
for S in 6 8 12; do echo "== S=$S" >> $out; timeout 300 python bench.py --config 3 --no-cpu-baseline --pair-streams $S >> $out 2>&1; done
