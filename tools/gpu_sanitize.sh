#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over small launches of
# every warp-specialised pipeline (tools/sanitize_cases.py)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1200 $CS --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/${TAG:-r02}_sanitize_$tool.txt 2>&1
  echo "rc=$?"
  tail -n 4 gpurun_out/${TAG:-r02}_sanitize_$tool.txt
done
