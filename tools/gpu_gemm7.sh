#!/bin/bash
timeout 300 python -m pytest tests/test_gemm.py -q -x 2>&1 | tail -1
ONLY="" timeout 300 python tools/gemm_bench.py 5 2>&1 | head -8
