#!/bin/bash
for m in 0 4 0x3f; do
echo "== NO_PAIR=$m"; MGLP_GEMM_NO_PAIR=$m timeout 600 python tools/profile_step.py bert 2>&1 | tail -24 | head -12
done
