#!/bin/bash
# attention tests + attention bench + GPT / ViT bench lines
timeout 600 python -m pytest tests/test_attention.py tests/test_presplit.py tests/test_parity.py -x -q 2>&1 | tail -2
python tools/attn_bench.py 10 2>&1 | grep "gpt\|vit"
for c in gpt vit; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c', round(d['value'],2), round(d['serial_ms_per_step'],1), d['clocks']['sm_mhz'])"; done
