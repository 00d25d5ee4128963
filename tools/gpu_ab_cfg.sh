#!/bin/bash
# same-box A/B of library builds (LIBS, _lib/libmglp_cuda_<x>.so) on whole
# MGRIT steps of the configs in CFGS, alternating; ENVS="VAR=a VAR=b" A/Bs an
# environment switch on the last build instead
mkdir -p gpurun_out
TAG=${TAG:-abc}
LIBS=${LIBS:-"A B"}
CFGS=${CFGS:-"gpt vit"}
run() {  # lib cfg env
  env $3 MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_$1.so timeout 900 python bench.py --config $2 --steps 3 --warmup 3 --no-extra --no-trainer --host-grads 0 --no-cpu-baseline 2>/dev/null | grep '^{"metric"' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1 $2 $3', round(d['value'],2), 'serial', round(d['serial_ms_per_step'],2), 'e2e', round(d['e2e']['value'],2), d['clocks']['sm_mhz'])" >> gpurun_out/${TAG}_ab.txt
}
for rep in 1 2; do
  for c in $CFGS; do
    if [ -n "$ENVS" ]; then
      for e in $ENVS; do run ${LIBS##* } $c $e; done
    else
      for lib in $LIBS; do run $lib $c ""; done
    fi
  done
done
cat gpurun_out/${TAG}_ab.txt
