#!/bin/bash
export ONLY=fwd MGLP_GEMM_PROF=1
echo "== pair"; timeout 300 python tools/gemm_bench.py 1 2>&1 | grep -v "^\s*$" | head -30
echo "== pair neither"; MGLP_DEBUG_GEMM=3 timeout 300 python tools/gemm_bench.py 1 2>&1 | head -30
