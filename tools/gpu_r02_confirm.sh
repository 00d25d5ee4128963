#!/bin/bash
# closing confirmation on one box: -m gpu suite, smoke, default bench line,
# per-config step breakdowns
mkdir -p gpurun_out
TAG=${TAG:-r02c}
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
for c in bert gpt vit; do timeout 600 python tools/profile_step.py $c > gpurun_out/${TAG}_breakdown_$c.txt 2>&1; done
tail -n 2 gpurun_out/${TAG}_gputest.log gpurun_out/${TAG}_smoke.log
tail -c 600 gpurun_out/${TAG}_bench.log
head -1 gpurun_out/${TAG}_breakdown_*.txt
