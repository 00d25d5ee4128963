"""One attention bench call (for ncu): python tools/attn_one.py G B H s dh causal mode reps"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09026_b200 import _native as N  # noqa: E402

G, B, H, s, dh, causal, mode, reps = (int(x) for x in sys.argv[1:9])
ms = C.c_float()
N.call("mglp_bench_attention", G, B, H, s, dh, causal, mode, reps, C.byref(ms))
print(f"{ms.value:.4f} ms")
