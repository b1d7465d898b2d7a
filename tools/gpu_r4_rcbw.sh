mkdir -p gpurun_out; rm -f gpurun_out/r4_rcbw2.log
for W in 6 30 100 1000 30 6; do
  echo "== c2 NRR_RCB_W=$W" >> gpurun_out/r4_rcbw2.log
  NRR_RCB_W=$W timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_rcbw2.log 2>&1
done
for W in 6 100; do
  echo "== c1 NRR_RCB_W=$W" >> gpurun_out/r4_rcbw2.log
  NRR_RCB_W=$W timeout 300 python bench.py --no-cpu-baseline --config 1 >> gpurun_out/r4_rcbw2.log 2>&1
  echo "== c4 NRR_RCB_W=$W" >> gpurun_out/r4_rcbw2.log
  NRR_RCB_W=$W timeout 600 python bench.py --no-cpu-baseline --config 4 --steps 10 >> gpurun_out/r4_rcbw2.log 2>&1
  echo "== c3 NRR_RCB_W=$W" >> gpurun_out/r4_rcbw2.log
  NRR_RCB_W=$W timeout 600 python bench.py --no-cpu-baseline --config 3 >> gpurun_out/r4_rcbw2.log 2>&1
done
