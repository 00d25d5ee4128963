#!/bin/bash
# full -m gpu suite with the parity report, smoke, default bench (round 2)
mkdir -p gpurun_out
MGLP_PARITY_REPORT=gpurun_out/r02_parity_report.json timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/r02_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02_smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/r02_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r02_bench.log
tail -n 3 gpurun_out/r02_gputest.log gpurun_out/r02_smoke.log gpurun_out/r02_bench.log
