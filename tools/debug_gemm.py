"""tcgen05 GEMM diagnostics: operand-major combinations and accumulation error."""
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09026_b200 import _native as N  # noqa: E402


def tf32_exact(x):
    return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)


def run(M, N_, K, a_mn, b_mn, pre, engine=0, exact=False, scaleB=1.0):
    torch.manual_seed(0)
    A = torch.randn((K, M) if a_mn else (M, K)).float().cuda()
    B = (torch.randn((K, N_) if b_mn else (N_, K)) * scaleB).float().cuda()
    if exact:
        A, B = tf32_exact(A), tf32_exact(B)
    C = torch.full((M, N_), float("nan"), device="cuda")
    N.call("mglp_test_gemm", 1, M, N_, K, A.data_ptr(), 0, M if a_mn else K, int(a_mn),
           B.data_ptr(), 0, N_ if b_mn else K, int(b_mn), int(pre), None, C.data_ptr(), 0, N_,
           engine)
    Ad = A.double().t() if a_mn else A.double()
    Bd = B.double().t() if b_mn else B.double()
    ref = Ad @ Bd.t()
    return ((C.double() - ref).abs().max() / ref.abs().max()).item(), \
        ((C.double() - ref).mean() / ref.abs().max()).item()


mode = sys.argv[1] if len(sys.argv) > 1 else "all"
if mode in ("all", "major"):
    for (M, Nn, K) in [(512, 512, 96), (300, 520, 100), (1024, 768, 768)]:
        for a_mn in (0, 1):
            for b_mn in (0, 1):
                e, _ = run(M, Nn, K, a_mn, b_mn, 1 - b_mn)
                print(f"pair M{M} N{Nn} K{K} a_mn={a_mn} b_mn={b_mn}: {e:.2e}", flush=True)
    for K in ():
        for a_mn in (0, 1):
            for b_mn in (0, 1):
                for pre in (0, 1):
                    e, _ = run(128, 256 if b_mn else 128, K, a_mn, b_mn, pre)
                    print(f"K{K} a_mn={a_mn} b_mn={b_mn} pre={pre}: {e:.2e}", flush=True)
if mode in ("all", "acc"):
    for K in (256, 1024, 2048, 4096):
        e0, b0 = run(256, 256, K, 0, 0, 1, exact=True)
        e1, b1 = run(256, 256, K, 0, 0, 1, exact=False)
        es, bs = run(256, 256, K, 0, 0, 0, engine=1)
        print(f"K{K}: tc exact-tf32 inputs {e0:.2e} (bias {b0:+.1e}) | tc general {e1:.2e} "
              f"(bias {b1:+.1e}) | simt fp32 {es:.2e} (bias {bs:+.1e})", flush=True)
