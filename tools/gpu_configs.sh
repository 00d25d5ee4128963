#!/bin/bash
# GPU check across every bench config (tests + one short bench line each).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
for c in tiny bert gpt vit mt; do
  echo "== $c"
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench_$c.err | tail -1 | tee gpurun_out/bench_$c.json
  tail -3 gpurun_out/bench_$c.err
done
timeout 600 python tools/profile_step.py bert 2>&1 | tail -24
