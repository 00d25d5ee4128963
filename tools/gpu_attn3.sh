#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/attn_bench.py 10 2>&1 | grep "bert\|mt"
A=MGLP_ATTN_P_FP32=1 B=MGLP_ATTN_P_FP32=0 bash tools/gpu_ab_env.sh
