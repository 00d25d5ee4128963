"""Device-timed fused attention (attn_tc.cu) on the hot-path head shapes
(C-ABI mglp_bench_attention). Usage: python tools/attn_bench.py [reps]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09026_b200 import _native as N  # noqa: E402

SHAPES = [  # name, G, B, H, s, dh, causal
    ("bert x16", 16, 32, 12, 128, 64, 0),
    ("bert x1", 1, 32, 12, 128, 64, 0),
    ("mt dec causal x16", 16, 32, 8, 128, 64, 1),
    ("tiny x4", 4, 8, 2, 32, 32, 0),
    ("gpt causal x32", 32, 8, 12, 512, 64, 1),
    ("vit x8", 8, 32, 12, 197, 64, 0),
]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
out = {}
MODES = [int(x) for x in os.environ.get("MODES", "0,1,2,3,4,5,13").split(",")]
for name, G, B, H, s, dh, causal in SHAPES:
    for bwd in MODES:
        ms = C.c_float()
        try:
            N.call("mglp_bench_attention", G, B, H, s, dh, causal, bwd, reps, C.byref(ms))
        except Exception as e:  # noqa: BLE001 (mode unsupported for the shape)
            print(f"{name} mode {bwd}: {e}")
            continue
        fl = (8.0 if (bwd & 3) == 1 else 4.0) * G * B * H * s * s * dh * (0.5 if causal else 1.0)
        key = f"{name} {['fwd', 'bwd', 'fwd noP', 'fwd noP Ohl'][bwd & 3]}{' hs' if bwd & 4 else ''}{' flash' if bwd & 8 else ''}"
        print(f"{key:24s} {ms.value:8.3f} ms  {fl / (ms.value * 1e-3) / 1e12:7.1f} TF/s", flush=True)
        out[key] = {"ms": ms.value, "tflops": fl / (ms.value * 1e-3) / 1e12}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/attn_bench{os.environ.get('TAG', '')}.json", "w"), indent=1)
