#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm.py -q -x 2>&1 | tail -2
echo "== default"; timeout 300 python tools/gemm_bench.py
echo "== no convert"; MGLP_DEBUG_GEMM=1 timeout 300 python tools/gemm_bench.py
echo "== no epilogue stores"; MGLP_DEBUG_GEMM=2 timeout 300 python tools/gemm_bench.py
echo "== neither"; MGLP_DEBUG_GEMM=3 timeout 300 python tools/gemm_bench.py
echo "== neither, 1 pass"; MGLP_DEBUG_SPLIT_PASSES=1 MGLP_DEBUG_GEMM=3 timeout 300 python tools/gemm_bench.py
