#!/bin/bash
timeout 300 python -m pytest tests/test_gemm.py -q -x 2>&1 | tail -1
for r in 5,3,4 4,3,5 6,3,3 3,3,6 4,4,4 5,4,3; do
  echo "== rings $r"; MGLP_GEMM_RINGS=$r ONLY=fwd timeout 300 python tools/gemm_bench.py 3 | head -7
done
