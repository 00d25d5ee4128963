mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 3000 --csv --log-file gpurun_out/r01_launches_bert.csv timeout 1200 python tools/profile_step.py bert > gpurun_out/r01_launches_stdout.txt 2>&1
