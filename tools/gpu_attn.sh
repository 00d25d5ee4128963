#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_attention.py -q -x 2>&1 | tail -15
timeout 300 python tools/attn_bench.py 2>&1 | tail -10
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
timeout 600 python tools/profile_step.py bert > gpurun_out/profile_bert.txt 2>&1; head -14 gpurun_out/profile_bert.txt
timeout 900 python bench.py --config bert --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
