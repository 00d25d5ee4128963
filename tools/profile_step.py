"""Per-shape device-time breakdown of one MGRIT fwd+bwd iteration (CUDA events
around every launch). Usage: python tools/profile_step.py [config]"""
import collections
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2601_09026_b200 import _native as N  # noqa: E402
from paper_2601_09026_b200.engine import SolveConfig, StackConfig  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bert"
cfg = bench.CONFIGS[name]
sc = StackConfig(kind=cfg["kind"], d=cfg["d"], heads=cfg["H"], ffn=cfg["ffn"], n_enc=cfg["n_enc"],
                 n_dec=cfg["n_dec"])
so = SolveConfig(coarsen=cfg["cf"], levels=cfg["levels"], fwd_iters=1, bwd_iters=1, warm_start=False)
h = C.c_void_p()
N.call("mglp_engine_create", C.byref(sc.desc()), C.byref(so.desc()), 0, C.byref(h))
N.call("mglp_engine_init_params", h, C.c_ulonglong(7), None)
ns = C.c_longlong()
N.call("mglp_engine_set_shape", h, cfg["B"], cfg["sx"], cfg["sy"], C.byref(ns))
z0 = torch.randn(ns.value, device="cuda") * 0.5
lam = torch.randn(ns.value, device="cuda")
lam0 = torch.zeros_like(z0)


def step():
    N.call("mglp_engine_forward_device", h, C.c_void_p(z0.data_ptr()))
    N.call("mglp_engine_backward_device", h, C.c_void_p(lam.data_ptr()), C.c_void_p(lam0.data_ptr()), 1)


step()
N.call("mglp_engine_sync", h)
N.call("mglp_engine_profile", h, 1)
step()
rows = np.zeros((20000, 8))
n = C.c_int()
N.call("mglp_engine_profile_dump", h, N.dptr(rows), 20000, C.byref(n))
rows = rows[:n.value]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
EPI = {0: "store", 1: "add2", 2: "gelu", 3: "final", 4: "gelu'", 5: "gacc"}
for cls, M, Nn, K, b, fl, ms, var in rows:
    key = (int(cls), int(M), int(Nn), int(K), int(b), int(var))
    agg[key][0] += 1
    agg[key][1] += ms
    agg[key][2] += fl
tot = rows[:, 6].sum()
print(f"{name}: {n.value} launches, {tot:.1f} ms in profiled kernels")
ROWK = {0: "row?", 1: "softmax", 2: "softmax_bwd", 3: "ln_fwd", 4: "ln_bwd", 5: "colred",
        6: "combine", 7: "copy", 8: "correct|pack"}
for key, (cnt, ms, fl) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:60]:
    cls, M, Nn, K, b, var = key
    if cls == 2:  # row kernel: (kind, cols, -, G); fl = HBM bytes
        gbs = fl / (ms * 1e-3) / 1e9 if ms > 0 else 0
        print(f"row   {ROWK.get(M, M):12s} cols {Nn:5d}   x{b:5d}  n={cnt:4d}  {ms:8.2f} ms "
              f"({100*ms/tot:5.1f}%)  {gbs:7.0f} GB/s")
        continue
    tf = fl / (ms * 1e-3) / 1e12 if ms > 0 else 0
    label = ["gemm", "other", "row"][cls]
    vs = ""
    if var >= 0:
        vs = EPI.get(var & 15, str(var & 15)) + ("" if not var & 16 else " Ahl") + \
            ("" if not var & 32 else " Bhl") + ("" if not var & 64 else " Amn") + ("" if not var & 128 else " Bmn")
    print(f"{label:5s} M{M:6d} N{Nn:5d} K{K:5d} x{b:5d} {vs:22s} n={cnt:4d}  {ms:8.2f} ms ({100*ms/tot:5.1f}%)  {tf:7.1f} TF/s")
