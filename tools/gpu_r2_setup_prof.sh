mkdir -p gpurun_out
python tools/setup_prof.py 2 > gpurun_out/r2_setup_prof.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_setup_launches.csv python tools/setup_prof.py 2 >> gpurun_out/r2_setup_prof.log 2>&1
echo rc=$? >> gpurun_out/r2_setup_prof.log
