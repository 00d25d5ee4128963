#!/bin/bash
# tests + BERT profile + BERT bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 600 python tools/profile_step.py ${CFG:-bert} > gpurun_out/profile_${CFG:-bert}.txt 2>&1; head -${NPROF:-16} gpurun_out/profile_${CFG:-bert}.txt
timeout 900 python bench.py --config ${CFG:-bert} --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_quick.json
python -c "import json;d=json.load(open('gpurun_out/bench_quick.json'));print('BENCH', d['config']['workload'], round(d['value'],2), 'serial', round(d['serial_ms_per_step'],1), 'e2e', round(d['e2e']['value'],2), 'frac', round(d['roofline']['frac'],3), d['clocks'])"
