# config 3 (batched pairs): side-by-side contexts sweep
mkdir -p gpurun_out
for S in 1 6; do
  timeout 900 python bench.py --config 3 --pairs 64 --pair-streams $S --no-cpu-baseline > gpurun_out/c3_s$S.log 2>&1
done
