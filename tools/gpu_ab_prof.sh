#!/bin/bash
# per-shape step profile (ln rows) + BERT bench for two library builds $LIBS
for lib in $LIBS $LIBS; do
  echo "== $lib"
  MGLP_LIB=paper_2601_09026_b200/_lib/$lib timeout 600 python tools/profile_step.py bert 2>&1 | grep "row" | head -4
  MGLP_LIB=paper_2601_09026_b200/_lib/$lib timeout 900 python bench.py --config bert --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bert', round(d['value'],2), d['clocks']['sm_mhz'])"
done
