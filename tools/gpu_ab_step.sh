#!/bin/bash
# A/B two library builds (libmglp_cuda_A.so / _B.so) on the BERT MGRIT step,
# the device serial sweep and the kernel breakdown, same box; then the GPU
# tests on the tree's build
mkdir -p gpurun_out
TAG=${TAG:-abs}
for lib in A B A B; do
  MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_$lib.so timeout 900 python bench.py --config bert --steps 5 --warmup 3 --no-extra --no-trainer --host-grads 0 --no-cpu-baseline 2>/dev/null | grep '^{"metric"' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$lib bench', round(d['value'],2), 'serial', round(d['serial_ms_per_step'],2), 'e2e', round(d['e2e']['value'],2), d['clocks']['sm_mhz'])" >> gpurun_out/${TAG}_ab.txt
  if [ -n "$BREAKDOWN" ]; then
    MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_$lib.so timeout 600 python tools/profile_step.py bert > gpurun_out/${TAG}_bert_$lib.txt 2>&1
    echo "$lib $(head -1 gpurun_out/${TAG}_bert_$lib.txt)" >> gpurun_out/${TAG}_ab.txt
    grep -E "$BREAKDOWN" gpurun_out/${TAG}_bert_$lib.txt | sed "s/^/$lib /" >> gpurun_out/${TAG}_ab.txt
  fi
done
[ -n "$NO_TESTS" ] && { cat gpurun_out/${TAG}_ab.txt; exit 0; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x ${TESTS_K:+-k "$TESTS_K"} > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
cat gpurun_out/${TAG}_ab.txt; tail -3 gpurun_out/${TAG}_tests.log
