set -x
ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 700 --csv --log-file gpurun_out/ncu_launches_bert.csv timeout 900 python tools/profile_step.py bert > gpurun_out/ncu_launches_stdout.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 10 -c 2 -o gpurun_out/ncu_gemm_pair timeout 1200 python tools/profile_step.py bert > gpurun_out/ncu_full_stdout.txt 2>&1
ls -la gpurun_out/
