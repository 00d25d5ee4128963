#!/bin/bash
# drain-epilogue diagnostics: mainloop speed with 3+3 vs 6+6 rings (epilogue
# stores skipped), and the per-role wait counters
for shape in "mlp_in  fwd A-hl" "mlp_out fwd A-hl" "qkv     fwd A-hl"; do
  for v in 0 1; do
    for dbg in 0 2; do
      echo "DRAIN=$v DEBUG=$dbg $(MGLP_GEMM_DRAIN=$v MGLP_DEBUG_GEMM=$dbg ONLY="$shape" timeout 120 python tools/gemm_bench.py 20 2>&1 | tail -1)"
    done
    echo "PROF DRAIN=$v $(MGLP_GEMM_DRAIN=$v MGLP_GEMM_PROF=1 ONLY="$shape" timeout 120 python tools/gemm_bench.py 1 2>&1 | grep gemm_prof | tail -1)"
  done
done
