#!/bin/bash
export ONLY=fwd
echo "== pair 4,4,4"; MGLP_GEMM_RINGS=4,4,4 timeout 300 python tools/gemm_bench.py 3 | head -5
echo "== pair 4,4,4 neither"; MGLP_DEBUG_GEMM=3 MGLP_GEMM_RINGS=4,4,4 timeout 300 python tools/gemm_bench.py 3 | head -5
echo "== 1cta"; MGLP_GEMM_NO_PAIR=0x3f MGLP_GEMM_RINGS=4,4,4 timeout 300 python tools/gemm_bench.py 3 | head -5
echo "== 1cta neither"; MGLP_DEBUG_GEMM=3 MGLP_GEMM_NO_PAIR=0x3f MGLP_GEMM_RINGS=4,4,4 timeout 300 python tools/gemm_bench.py 3 | head -5
echo "== 1cta neither 1pass"; MGLP_DEBUG_SPLIT_PASSES=1 MGLP_DEBUG_GEMM=3 MGLP_GEMM_NO_PAIR=0x3f MGLP_GEMM_RINGS=4,4,4 timeout 300 python tools/gemm_bench.py 3 | head -5
