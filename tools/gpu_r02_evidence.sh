#!/bin/bash
# round-2 evidence on one box: full -m gpu suite (+ parity report), smoke,
# default bench line, ncu launch list of one BERT iteration
mkdir -p gpurun_out
TAG=${TAG:-r02}
MGLP_PARITY_REPORT=gpurun_out/${TAG}_parity_report.json timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/${TAG}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
if [ -z "${NO_NCU}" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/${TAG}_launches_bert.csv timeout 1200 python tools/profile_step.py bert \
    > gpurun_out/${TAG}_launches_stdout.txt 2>&1
fi
tail -n 3 gpurun_out/${TAG}_gputest.log gpurun_out/${TAG}_smoke.log
tail -c 3000 gpurun_out/${TAG}_bench.log
