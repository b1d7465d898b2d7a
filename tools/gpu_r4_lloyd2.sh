mkdir -p gpurun_out; rm -f gpurun_out/r4_lloyd2.log
for L in 0 16; do for C in 10 17 25; do
  [ "$L" = "0" ] && [ "$C" != "17" ] && continue
  echo "== c2 NRR_LLOYD=$L CAP=$C" >> gpurun_out/r4_lloyd2.log
  NRR_LLOYD=$L NRR_LLOYD_CAP=$C timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_lloyd2.log 2>&1
  NRR_LLOYD=$L NRR_LLOYD_CAP=$C timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/r4_lloyd2.log 2>&1
done; done
