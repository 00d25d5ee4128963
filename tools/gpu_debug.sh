python tools/debug_gemm.py all 2>&1 | tail -40
echo "== passes=1"
MGLP_DEBUG_TF32_PASSES=1 python tools/debug_gemm.py acc 2>&1 | tail -6
python tools/debug_parity.py enc_small 2>&1 | head -30
