#!/bin/bash
timeout 300 python -m pytest tests/test_gemm.py -q -x 2>&1 | tail -2 || exit 1
echo "== gemm"; timeout 300 python tools/gemm_bench.py
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 600 python tools/profile_step.py bert 2>&1 | tail -24
timeout 900 python bench.py --config bert --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
