#!/bin/bash
# Full GPU check: tests, parity report, every bench config (N=1)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 900 python tools/parity_report.py > gpurun_out/parity_report.log 2>&1
for c in tiny bert gpt vit mt; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 2>gpurun_out/bench_$c.err | tail -1 > gpurun_out/bench_$c.json
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', round(d['value'],1), 'serial', round(d['serial_ms_per_step'],1), 'probe', round(d['monitor_probe_ms_per_step'],1), 'frac', round(d['roofline']['frac'],3), 'cpu', d.get('cpu_baseline'))" 2>&1 | tail -1
done
timeout 600 python tools/profile_step.py bert > gpurun_out/profile_bert.txt 2>&1
