"""Timeline of CTA 0 of the flash dK/dV kernel (MGLP_FLASH_TRACE build):
MGLP_LIB=paper_2601_09026_b200/_lib/libmglp_cuda_trace.so python tools/flash_trace.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09026_b200 import _native as N  # noqa: E402

ms = C.c_float()
N.call("mglp_bench_attention", 32, 8, 12, 512, 64, 1, 13, 1, C.byref(ms))
buf = (C.c_longlong * 4096)()
N.lib().mglp_debug_flash_trace(buf, 4096)
t0 = buf[6]
names = ["mma:Q ready", "mma:S issue", "mma:grads issue(prev)", "cmp:wait S", "cmp:S ready", "cmp:P done", "ld:Q issue"]
for step in range(40):
    row = [buf[8 * step + k] - t0 if buf[8 * step + k] else None for k in range(7)]
    print(step, "  ".join(f"{n.split(':')[1][:10]:>10s}={v if v is not None else '-':>8}" for n, v in zip(names, row)))
print("problem   KV issue   MMA KV ready   epi start   epi end   (cycles from the first Q issue)")
for p in range(8):
    row = [buf[2048 + 4 * p + k] - t0 if buf[2048 + 4 * p + k] else None for k in (0, 3, 1, 2)]
    print(p, "  ".join(f"{v if v is not None else '-':>10}" for v in row))
