mkdir -p gpurun_out
for f in 100 10 1; do
  NRR_PCG_TRUE_FACTOR=$f timeout 600 python tools/diag_rtol.py 1e-12,1e-13,1e-14 >> gpurun_out/rtol.log 2>&1
  for r in 1e-12 1e-13 1e-14; do
    echo "factor $f rtol $r" >> gpurun_out/rtol_bench.log
    NRR_PCG_TRUE_FACTOR=$f timeout 300 python bench.py --no-cpu-baseline --steps 30 --pcg-rtol $r 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['pcg_iterations_per_step'], d['kernel_ms_per_step'])
    else: print(l.rstrip())" >> gpurun_out/rtol_bench.log
  done
done
