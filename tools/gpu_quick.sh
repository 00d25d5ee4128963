#!/bin/bash
# quick check: selected GPU tests (PYTEST_SEL), then the per-config breakdowns
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout ${PYT:-900} python -m pytest ${PYTEST_SEL:-tests/test_attention.py} -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_tests.log
tail -n 15 gpurun_out/${TAG}_tests.log
for c in ${CONFIGS:-bert}; do
  timeout 600 python tools/profile_step.py $c > gpurun_out/${TAG}_breakdown_$c.txt 2>&1
  head -14 gpurun_out/${TAG}_breakdown_$c.txt
done
if [ -n "${BENCH}" ]; then timeout 900 python bench.py ${BENCH_ARGS} 2>/dev/null | tail -1 > gpurun_out/${TAG}_bench.json; head -c 600 gpurun_out/${TAG}_bench.json; fi
