#!/bin/bash
# A/B of env settings on the same box: BERT bench value
for env in "X=0" "MGLP_GEMM_RINGS=3,3,6" "X=0" "MGLP_GEMM_RINGS=3,3,6"; do
  v=$(env $env timeout 900 python bench.py --config bert --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), d['clocks']['sm_mhz'])")
  echo "$env -> $v"
done
