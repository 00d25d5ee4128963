#!/bin/bash
# diagnostics of the converter-free pair GEMM: epilogue skipped (MGLP_DEBUG_GEMM=2),
# 1-pass (MGLP_DEBUG_SPLIT_PASSES=1), all units on the same L2-resident tiles
# (MGLP_DEBUG_GEMM=4), and the per-role wait counters
for o in "mlp_in  fwd A-hl" "mlp_out fwd A-hl" "o       fwd A-hl"; do
  for env in "X=0" "MGLP_DEBUG_GEMM=2" "MGLP_DEBUG_GEMM=6" "MGLP_DEBUG_SPLIT_PASSES=1 MGLP_DEBUG_GEMM=2" "MGLP_DEBUG_SPLIT_PASSES=1 MGLP_DEBUG_GEMM=6"; do
    echo "$env: $(env $env ONLY="$o" timeout 300 python tools/gemm_bench.py 10 2>&1 | tail -1)"
  done
done
