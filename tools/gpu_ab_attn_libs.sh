#!/bin/bash
# A/B of two library builds on the long-attention kernels, then attention tests on B
mkdir -p gpurun_out
for lib in A B A B; do
  echo "== $lib" >> gpurun_out/abattn.txt
  MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_$lib.so MODES=13,12 timeout 300 python tools/attn_bench.py 5 2>&1 | grep -E "gpt|vit" >> gpurun_out/abattn.txt
done
MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_B.so timeout 900 python -m pytest tests/test_attention.py -q -x -p no:cacheprovider > gpurun_out/abattn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/abattn_tests.log
cat gpurun_out/abattn.txt; tail -3 gpurun_out/abattn_tests.log
