# config 3 A/B: PCG on a greatest-priority stream (default) vs the context stream
mkdir -p gpurun_out
for i in 1 2 3 4; do
  timeout 240 python bench.py --config 3 --no-cpu-baseline > gpurun_out/c3ab_p$i.log 2>&1; echo "p$i rc=$?" >> gpurun_out/c3ab_summary.log
  NRR_NO_PCG_PRIORITY=1 timeout 240 python bench.py --config 3 --no-cpu-baseline > gpurun_out/c3ab_n$i.log 2>&1; echo "n$i rc=$?" >> gpurun_out/c3ab_summary.log
done
