#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm.py -q -x 2>&1 | tail -3
echo "== default"; timeout 300 python tools/gemm_bench.py
echo "== no pair"; MGLP_GEMM_NO_PAIR=1 timeout 300 python tools/gemm_bench.py
echo "== 1 pass"; MGLP_DEBUG_SPLIT_PASSES=1 timeout 300 python tools/gemm_bench.py
ONLY="mlp_out fwd" timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/ncu_f16_pair -f python tools/gemm_bench.py 1 > gpurun_out/ncu_f16_stdout.txt 2>&1
ONLY="attn S" timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/ncu_f16_single -f python tools/gemm_bench.py 1 >> gpurun_out/ncu_f16_stdout.txt 2>&1
tail -3 gpurun_out/ncu_f16_stdout.txt
