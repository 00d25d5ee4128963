#!/bin/bash
# engine parity on the attention paths, then GPT / ViT with and without the stored dS tiles
timeout 600 python -m pytest tests/test_attention.py tests/test_presplit.py -x -q 2>&1 | tail -3
for c in vit gpt; do
  for env in "MGLP_LONG_DS=0" "MGLP_LONG_DS=1"; do
    v=$(env $env timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), round(d['serial_ms_per_step'],1), d['clocks']['sm_mhz'])")
    echo "$c $env -> $v"
  done
done
