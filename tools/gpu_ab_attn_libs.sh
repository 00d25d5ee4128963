#!/bin/bash
# A/B of library builds (LIBS="A B ...": _lib/libmglp_cuda_<x>.so) on the
# long-attention kernels, then the attention tests (and REPEAT extra runs of
# the many-problem flash backward test) on the last build
mkdir -p gpurun_out
LIBS=${LIBS:-"A B"}
for rep in 1 2; do
  for lib in $LIBS; do
    echo "== $lib" >> gpurun_out/abattn.txt
    MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_$lib.so MODES=13,12 timeout 300 python tools/attn_bench.py 5 2>&1 | grep -E "gpt|vit" >> gpurun_out/abattn.txt
  done
done
last=${LIBS##* }
MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_$last.so timeout 900 python -m pytest tests/test_attention.py -q -x -p no:cacheprovider > gpurun_out/abattn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/abattn_tests.log
for i in $(seq 1 ${REPEAT:-0}); do
  MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_$last.so timeout 300 python -m pytest tests/test_attention.py -q -x -p no:cacheprovider -k flash_backward > /dev/null 2>&1 || echo "repeat $i FAILED rc=$?" >> gpurun_out/abattn_tests.log
done
[ -n "$TRACE" ] && MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_trace.so timeout 120 python tools/flash_trace.py > gpurun_out/ftrace.txt 2>&1
cat gpurun_out/abattn.txt; tail -4 gpurun_out/abattn_tests.log
