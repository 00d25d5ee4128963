#!/bin/bash
# TMEM-drain pair GEMM: correctness (GEMM + parity tests) and A/B against the
# TMEM-held epilogue on the converter-free shapes and the BERT step
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm.py tests/test_parity.py tests/test_deep_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -n 5
for v in 1 0; do
  for shape in "mlp_in  fwd A-hl" "mlp_out fwd A-hl" "qkv     fwd A-hl" "o       fwd A-hl" "mlp_out dgrad gelu'"; do
    echo "DRAIN=$v $(MGLP_GEMM_DRAIN=$v ONLY="$shape" timeout 120 python tools/gemm_bench.py 20 2>&1 | tail -1)"
  done
done
for v in 1 0 1; do
  echo "DRAIN=$v bench: $(MGLP_GEMM_DRAIN=$v timeout 600 python bench.py --steps 10 --no-extra --no-trainer --host-grads 0 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["roofline"]["achieved"], d["clocks"]["sm_mhz"])')"
done
