mkdir -p gpurun_out
out=gpurun_out/r2_sweep3.log; : > $out
for C in 216 500; do
  echo "== c2 H=1.0 CELLS=$C" >> $out; NRR_NN_GRID_H=1.0 NRR_NN_GRID_CELLS=$C timeout 300 python bench.py --no-cpu-baseline --steps 20 >> $out 2>&1
  echo "== c4 H=1.0 CELLS=$C" >> $out; NRR_NN_GRID_H=1.0 NRR_NN_GRID_CELLS=$C timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> $out 2>&1
done
echo "== c2 default" >> $out; timeout 300 python bench.py --no-cpu-baseline --steps 20 >> $out 2>&1
for S in 9 10 6 9 12; do echo "== c3 S=$S" >> $out; timeout 300 python bench.py --config 3 --no-cpu-baseline --pair-streams $S >> $out 2>&1; done
