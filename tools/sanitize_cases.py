"""Small launches of every warp-specialised tcgen05 pipeline for
compute-sanitizer (racecheck / synccheck / memcheck): the 1-CTA and CTA-pair
GEMMs (converted and pre-split operands; the TMEM-drain epilogue), the fused
s=128 attention and the long (s=256, causal) attention, and one tiny MGRIT
fwd+bwd through the engine. Usage: python tools/sanitize_cases.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_attention as TA  # noqa: E402
import test_gemm as TG  # noqa: E402

for shape in [(1, 128, 128, 64, False, False, True), (1, 256, 256, 64, False, False, True),
              (1, 256, 256, 64, True, True, False), (1, 256, 256, 96, False, False, True)]:
    G, M, N_, K, amn, bmn, pre = shape
    c, ref = TG.run(G, M, N_, K, amn, bmn, pre, engine=0, bias=True)
    print("gemm", shape, TG.relerr(c, ref), flush=True)
import ctypes as C  # noqa: E402
from paper_2601_09026_b200 import _native as N  # noqa: E402
ms = C.c_float()
# converter-free pair GEMM (pre-split A and B): the TMEM-drain epilogue
N.call("mglp_bench_gemm", 1, 256, 512, 64, 0, 0, 3, 0, 1, C.byref(ms))
print("gemm drain ok", flush=True)
for (B, H, s, causal) in [(1, 1, 128, False), (1, 1, 256, True)]:
    out = TA.run(B, H, s, s, 64, causal)
    print("attention", (B, H, s, causal), "ok", flush=True)
# single-pass long attention with every operand pre-split (attn_flash.cu):
# several problems per CTA of the dK/dV kernel (steps chained across
# problems), a ragged 197-token shape and a 512-token causal one
for (B, H, s, causal) in [(2, 2, 197, False), (1, 2, 512, True), (1, 1, 256, True)]:
    got, ref = TA.run(B, H, s, s, 64, int(causal) | 4 | 8, seed=9)
    print("flash attention", (B, H, s, causal),
          [round(TA.relerr(a, b), 8) for n, a, b in zip("OPQKV", got, ref) if n != "P"], flush=True)
import __graft_entry__ as GE  # noqa: E402
GE.smoke()
print("engine ok", flush=True)
