#!/bin/bash
# A/B two library builds (libmglp_cuda_A.so / _B.so) on the s = 128 attention
# kernels and the BERT step, same box; then the attention tests on the build
mkdir -p gpurun_out
TAG=${TAG:-ab}
for lib in A B A B; do
  echo "== $lib" >> gpurun_out/${TAG}_ab.txt
  MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_$lib.so MODES=0,5 timeout 300 python tools/attn_bench.py 20 2>&1 | grep "bert x16" >> gpurun_out/${TAG}_ab.txt
  MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_$lib.so timeout 600 python tools/profile_step.py bert > gpurun_out/${TAG}_bert_$lib.txt 2>&1
  head -1 gpurun_out/${TAG}_bert_$lib.txt >> gpurun_out/${TAG}_ab.txt
  grep "M  -128 N  128 K   64 x 6144" gpurun_out/${TAG}_bert_$lib.txt >> gpurun_out/${TAG}_ab.txt
done
timeout 1200 python -m pytest tests/test_attention.py tests/test_variants_bitwise.py -q -p no:cacheprovider -x > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
cat gpurun_out/${TAG}_ab.txt; tail -3 gpurun_out/${TAG}_tests.log
