#!/bin/bash
for c in gpt vit mt; do
  timeout 900 python tools/profile_step.py $c > gpurun_out/profile_$c.txt 2>&1; head -14 gpurun_out/profile_$c.txt
done
