#!/bin/bash
# quick GEMM check first (short timeout: a pipeline deadlock must not hang the box)
timeout 300 python -m pytest tests/test_gemm.py -q -x 2>&1 | tail -15 || exit 1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -8
timeout 900 python tools/parity_report.py 2>&1 | tail -8
timeout 600 python tools/profile_step.py bert > gpurun_out/profile_bert.txt 2>&1; head -12 gpurun_out/profile_bert.txt
timeout 900 python bench.py --config bert --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
