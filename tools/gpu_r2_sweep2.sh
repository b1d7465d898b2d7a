mkdir -p gpurun_out
out=gpurun_out/r2_sweep2.log; : > $out
for H in 0.7 0.85 1.0; do for C in 1000 3000; do
  echo "== c2 H=$H CELLS=$C" >> $out
  NRR_NN_GRID_H=$H NRR_NN_GRID_CELLS=$C timeout 300 python bench.py --no-cpu-baseline --steps 20 >> $out 2>&1
done; done
for H in 0.7 1.0; do echo "== c4 H=$H CELLS=3000" >> $out; NRR_NN_GRID_H=$H NRR_NN_GRID_CELLS=3000 timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> $out 2>&1; done
for B in 8 16 32; do echo "== aa blocks $B" >> $out; NRR_AA_BLOCKS=$B timeout 300 python bench.py --no-cpu-baseline --steps 20 >> $out 2>&1; done
for S in 6 7 8 9; do echo "== c3 S=$S" >> $out; timeout 300 python bench.py --config 3 --no-cpu-baseline --pair-streams $S >> $out 2>&1; done
