#!/bin/bash
# GEMM power/clock diagnostics: each variant runs ~3 s while nvidia-smi samples
# clocks and power; MGLP_DEBUG_GEMM=2 skips the epilogue stores
mkdir -p gpurun_out
run() {
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > gpurun_out/pw.csv &
  P=$!
  sleep 0.5
  out=$(env $1 ONLY="$2" timeout 120 python tools/gemm_bench.py $3 2>&1 | tail -1)
  kill $P; wait $P 2>/dev/null
  stats=$(python - <<'PY'
import statistics
r=[l.split(',') for l in open('gpurun_out/pw.csv') if l.strip()]
c=[float(x[0]) for x in r]; p=[float(x[1]) for x in r]
c=c[len(c)//4:]; p=p[len(p)//4:]
print(f"sm {statistics.median(c):.0f} MHz  power {statistics.median(p):.0f} W (n={len(c)})")
PY
)
  echo "$1 | $out | $stats"
}
for shape in "mlp_in  fwd A-hl" "mlp_out fwd A-hl" "o       fwd A-hl" "wgrad w_in" "mlp_out dgrad gelu'"; do
  run "X=0" "$shape" 2000
  run "MGLP_DEBUG_GEMM=2" "$shape" 2000
done
