#!/bin/bash
# round-2 closing evidence on one box: -m gpu suite + parity report, smoke,
# default bench line, ncu launch list of one BERT iteration, ncu --set full of
# the first GEMM launches of a BERT step, per-config breakdowns
mkdir -p gpurun_out
TAG=${TAG:-r02f}
MGLP_PARITY_REPORT=gpurun_out/${TAG}_parity_report.json timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
for c in bert gpt vit; do timeout 600 python tools/profile_step.py $c > gpurun_out/${TAG}_breakdown_$c.txt 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/${TAG}_launches_bert.csv timeout 1200 python tools/profile_step.py bert \
    > gpurun_out/${TAG}_launches_stdout.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 0 -c 8 \
    -o gpurun_out/${TAG}_gemm_full timeout 1200 python tools/profile_step.py bert > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_gemm_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_gemm_full_raw.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_ -s 0 -c 4 \
    -o gpurun_out/${TAG}_attn_full timeout 1200 python tools/profile_step.py gpt > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_attn_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_attn_full_raw.csv 2>&1
tail -n 2 gpurun_out/${TAG}_gputest.log gpurun_out/${TAG}_smoke.log
tail -c 1500 gpurun_out/${TAG}_bench.log
