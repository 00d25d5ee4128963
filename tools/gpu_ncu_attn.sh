#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-a}
ncu --set full --clock-control none --import-source on -k regex:${KRE:-attn_} -s ${SKIP:-2} -c ${COUNT:-1} \
    -o gpurun_out/ncu_attn_$TAG timeout 600 python tools/attn_bench.py 2 > gpurun_out/ncu_attn_$TAG.stdout 2>&1
ncu -i gpurun_out/ncu_attn_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_attn_${TAG}_details.csv 2>&1
ncu -i gpurun_out/ncu_attn_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_attn_${TAG}_sass.csv 2>&1
ncu -i gpurun_out/ncu_attn_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_attn_${TAG}_raw.csv 2>&1
