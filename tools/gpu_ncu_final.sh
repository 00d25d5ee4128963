#!/bin/bash
# Evidence for the judge: (1) launch list of one BERT iteration (second step of
# tools/profile_step.py; cold-cache, serialised per-launch times -> compare
# SHARES), (2) one --set full capture of the dominant GEMM (pair kernel,
# MLP-in family) and of the fused attention kernels.
mkdir -p gpurun_out
TAG=${TAG:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-0} -c ${COUNT:-3000} --csv \
    --log-file gpurun_out/${TAG}_launches_bert.csv timeout 1200 python tools/profile_step.py bert \
    > gpurun_out/${TAG}_launches_stdout.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s ${GSKIP:-10} -c 6 \
    -o gpurun_out/${TAG}_gemm_full timeout 1200 python tools/profile_step.py bert > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_gemm_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_gemm_full_raw.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_ -s 2 -c 2 \
    -o gpurun_out/${TAG}_attn_full timeout 1200 python tools/profile_step.py bert > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_attn_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_attn_full_raw.csv 2>&1
rm -f gpurun_out/${TAG}_gemm_full.ncu-rep.bak
ls -la gpurun_out | tail -8
