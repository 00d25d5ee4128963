#!/bin/bash
# per-shape/variant breakdown (CUDA events) of one iteration per config, and
# one ncu --set full capture of the first GEMM launches of a BERT step
mkdir -p gpurun_out
TAG=${TAG:-r02p}
for c in ${CONFIGS:-bert gpt vit}; do
  timeout 600 python tools/profile_step.py $c > gpurun_out/${TAG}_breakdown_$c.txt 2>&1
done
if [ -n "${NCU}" ]; then
ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-gemm_tc_kernel} -s ${GSKIP:-0} -c ${GCOUNT:-8} \
    -o gpurun_out/${TAG}_full timeout 1200 python tools/profile_step.py bert > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_raw.csv 2>&1
fi
head -45 gpurun_out/${TAG}_breakdown_*.txt
