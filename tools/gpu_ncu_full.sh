#!/bin/bash
# One ncu --set full capture of the first GEMM family launches of a BERT step
# (QKV, attention S/PV, O-proj, MLP-in, MLP-out), plus a raw CSV export.
mkdir -p gpurun_out
TAG=${1:-cur}
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s ${SKIP:-0} -c ${COUNT:-8} \
    -o gpurun_out/ncu_full_$TAG timeout 1200 python tools/profile_step.py bert > gpurun_out/ncu_full_$TAG.stdout 2>&1
ncu -i gpurun_out/ncu_full_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_full_${TAG}_raw.csv 2>&1
ncu -i gpurun_out/ncu_full_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_full_${TAG}_details.csv 2>&1
ls -la gpurun_out/
