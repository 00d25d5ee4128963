#!/bin/bash
# one ncu --set full capture of a kernel (regex NCU_K) launched by CMD; raw + source CSVs
mkdir -p gpurun_out
TAG=${TAG:-k}
ncu --set full --clock-control none --import-source on -k regex:${NCU_K} -s ${SKIP:-0} -c ${COUNT:-1} \
    -o gpurun_out/${TAG} timeout 600 ${CMD} > gpurun_out/${TAG}_stdout.txt 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page details > gpurun_out/${TAG}_details.txt 2>&1
tail -5 gpurun_out/${TAG}_stdout.txt
grep -E "Duration|Throughput|Tensor|Issue|Warp Cycles|Eligible|Registers|Occupancy|No Eligible|Active Warps" gpurun_out/${TAG}_details.txt | head -40
