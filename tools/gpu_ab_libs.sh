#!/bin/bash
# A/B builds of the library on one box: $LIBS (paper_2601_09026_b200/_lib/<name>), optional env $ENVS per lib
CFG=${CFG:-bert}
for lib in $LIBS $LIBS; do
  v=$(MGLP_LIB=paper_2601_09026_b200/_lib/$lib timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), round(d['serial_ms_per_step'],1), d['clocks']['sm_mhz'])")
  echo "$CFG $lib -> $v"
done
