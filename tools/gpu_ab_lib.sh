#!/bin/bash
# A/B two builds of the library on the same box: gemm_bench + BERT bench
for lib in libmglp_cuda_nopf.so libmglp_cuda_pf.so libmglp_cuda_nopf.so libmglp_cuda_pf.so; do
  echo "== $lib"
  MGLP_LIB=paper_2601_09026_b200/_lib/$lib timeout 300 python tools/gemm_bench.py 5 2>&1 | head -6
  MGLP_LIB=paper_2601_09026_b200/_lib/$lib timeout 900 python bench.py --config bert --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BERT', round(d['value'],2), d['clocks']['sm_mhz'])"
done
