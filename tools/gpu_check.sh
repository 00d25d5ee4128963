set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gemm.py -x -q 2>&1 | tail -30
MGLP_LIB=$PWD/paper_2601_09026_b200/_lib/libmglp_cuda_simtref.so timeout 900 python -m pytest tests/test_parity.py -x -q 2>&1 | tail -30
timeout 900 python -m pytest tests/test_parity.py -q 2>&1 | tail -30
