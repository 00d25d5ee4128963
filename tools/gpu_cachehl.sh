#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/gemm_bench.py 10 2>&1 | grep wgrad
for i in 1 2; do timeout 900 python bench.py --config bert --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bert', round(d['value'],2), round(d['serial_ms_per_step'],1), d['clocks']['sm_mhz'])"; done
