#!/bin/bash
# A/B an env setting on the same box: BERT (or $CFG) bench value
for env in "${A:-X=0}" "${B:-X=1}" "${A:-X=0}" "${B:-X=1}"; do
  v=$(env $env timeout 900 python bench.py --config ${CFG:-bert} --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), round(d['serial_ms_per_step'],1), d['clocks']['sm_mhz'])")
  echo "$env -> $v"
done
