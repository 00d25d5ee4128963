#!/bin/bash
# Round evidence on one B200: GPU tests, measured parity, a bench line per
# config (-> profiles/<tag>_bench_configs.jsonl), the per-shape step profile,
# and the ncu launch list + --set full captures (tools/ncu_summarize.py).
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/${TAG}_gpu_tests.txt
timeout 900 python tools/parity_report.py > gpurun_out/${TAG}_parity_stdout.txt 2>&1
: > gpurun_out/${TAG}_bench_configs.jsonl
for c in tiny bert gpt vit mt; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 2>gpurun_out/bench_$c.err | tail -1 \
    >> gpurun_out/${TAG}_bench_configs.jsonl
done
timeout 600 python tools/profile_step.py bert > gpurun_out/${TAG}_bert_step_breakdown.txt 2>&1
TAG=$TAG bash tools/gpu_ncu_final.sh > /dev/null 2>&1
ls -la gpurun_out | tail -12
