#!/bin/bash
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for c in ${CFGS:-gpt vit}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_$c.json
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('BENCH', '$c', round(d['value'],1), 'serial', round(d['serial_ms_per_step'],1), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
