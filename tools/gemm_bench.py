"""Device-timed throughput of the tensor-core GEMM on the hot-path shapes
(C-ABI mglp_bench_gemm). Usage: python tools/gemm_bench.py [reps]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09026_b200 import _native as N  # noqa: E402

SHAPES = [  # (name, G, M, N, K, a_mn, b_mn, presplit[, epilogue kind])
    ("mlp_in  fwd", 16, 4096, 3072, 768, 0, 0, 1),
    ("mlp_in  fwd A-hl", 16, 4096, 3072, 768, 0, 0, 3),
    ("mlp_in  fwd gelu", 16, 4096, 3072, 768, 0, 0, 1, 2),
    ("mlp_out dgrad gelu'", 16, 4096, 3072, 768, 0, 1, 1, 4),
    ("mlp_out fwd", 16, 4096, 768, 3072, 0, 0, 1),
    ("mlp_out fwd A-hl", 16, 4096, 768, 3072, 0, 0, 3),
    ("qkv     fwd", 16, 4096, 2304, 768, 0, 0, 1),
    ("qkv     fwd A-hl", 16, 4096, 2304, 768, 0, 0, 3),
    ("o       fwd", 16, 4096, 768, 768, 0, 0, 1),
    ("o       fwd A-hl", 16, 4096, 768, 768, 0, 0, 3),
    ("mlp_in  dgrad", 16, 4096, 768, 3072, 0, 1, 1),
    ("wgrad w_in", 16, 3072, 768, 4096, 1, 1, 0),
    ("attn S", 6144, 128, 128, 64, 0, 0, 0),
    ("attn PV", 6144, 128, 64, 128, 0, 1, 0),
    ("square 8192", 1, 8192, 8192, 8192, 0, 0, 1),
]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
out = {}
only = os.environ.get("ONLY")
for name, G, M, Nn, K, amn, bmn, pre, *epi in SHAPES:
    if only and only not in name:
        continue
    ms = C.c_float()
    N.call("mglp_bench_gemm", G, M, Nn, K, amn, bmn, pre, epi[0] if epi else 0, reps, C.byref(ms))
    tf = 2.0 * G * M * Nn * K / (ms.value * 1e-3) / 1e12
    print(f"{name:20s} G={G:5d} M={M:5d} N={Nn:5d} K={K:5d}  {ms.value:8.3f} ms  {tf:7.1f} TF/s",
          flush=True)
    out[name] = {"ms": ms.value, "tflops": tf}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/gemm_bench{os.environ.get('TAG', '')}.json", "w"), indent=1)
