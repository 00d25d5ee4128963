#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
A=MGLP_NO_CACHE_HL=1 B=MGLP_NO_CACHE_HL=0 bash tools/gpu_ab_env.sh
