#!/bin/bash
# ncu --set full of the attention kernels inside one step: BERT (s = 128 fused)
# and GPT-2 (single-pass forward / backward)
mkdir -p gpurun_out
TAG=${TAG:-r02a}
ncu --set full --clock-control none -k regex:"attn_fwd_kernel" -s 0 -c 2 \
    -o gpurun_out/${TAG}_bertf timeout 900 python tools/profile_step.py bert > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"attn_bwd_kernel" -s 0 -c 2 \
    -o gpurun_out/${TAG}_bertb timeout 900 python tools/profile_step.py bert > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"attn_fwd_flash" -s 0 -c 2 \
    -o gpurun_out/${TAG}_gptf timeout 900 python tools/profile_step.py gpt > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"kv_flash|q_flash|flash_rowdot" -s 0 -c 3 \
    -o gpurun_out/${TAG}_gptb timeout 900 python tools/profile_step.py gpt > /dev/null 2>&1
for k in bertf bertb gptf gptb; do
  ncu -i gpurun_out/${TAG}_$k.ncu-rep --page raw --csv > gpurun_out/${TAG}_${k}_raw.csv 2>&1
  rm -f gpurun_out/${TAG}_$k.ncu-rep
done
ls -la gpurun_out | grep ${TAG}
