# config 3: default (cooperative grids side by side, budget fix) x5, then the cluster PCG at 6/9 streams
mkdir -p gpurun_out
out=gpurun_out/r2_c3.log
: > $out
for i in 1 2 3 4 5; do
  echo "== default run $i" >> $out
  timeout 180 python bench.py --config 3 --no-cpu-baseline >> $out 2>&1; echo "rc=$?" >> $out
done
for S in 6 9 12; do
  echo "== cluster S=$S" >> $out
  NRR_PCG=cluster timeout 180 python bench.py --config 3 --no-cpu-baseline --pair-streams $S >> $out 2>&1; echo "rc=$?" >> $out
done
