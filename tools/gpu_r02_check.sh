#!/bin/bash
# new GPU tests (monitor, integration, lambda scale, range) + sanitizers + bench A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_integration.py tests/test_monitor.py tests/test_lambda_scale.py tests/test_range.py tests/test_parity.py tests/test_dist.py -m gpu -q -p no:cacheprovider > gpurun_out/r02_check.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_check.log
tail -n 15 gpurun_out/r02_check.log
bash tools/gpu_sanitize.sh
for v in 1 0; do
  echo "DRAIN=$v bench: $(MGLP_GEMM_DRAIN=$v timeout 600 python bench.py --steps 10 --no-extra --no-trainer --host-grads 0 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["roofline"]["achieved"], d["clocks"]["sm_mhz"])')"
done
