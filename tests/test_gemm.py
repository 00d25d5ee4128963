"""tcgen05 kind::tf32 x3 GEMM (the product kernel) against an fp64 torch
reference and the fp32 CUDA-core reference kernel, through the C-ABI test hook."""
import ctypes as C
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
from paper_2601_09026_b200 import _native as N  # noqa: E402

pytestmark = pytest.mark.gpu


def run(G, M, N_, K, a_mn, b_mn, presplit, engine, bias=False, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    A = torch.randn(G, *( (K, M) if a_mn else (M, K) ), generator=g).float().cuda()
    B = (torch.randn(G, *( (K, N_) if b_mn else (N_, K) ), generator=g) * 0.05).float().cuda()
    bv = torch.randn(N_, generator=g).float().cuda() if bias else None
    Cm = torch.full((G, M, N_), float("nan"), device="cuda")
    lda = M if a_mn else K
    ldb = N_ if b_mn else K
    N.call("mglp_test_gemm", G, M, N_, K, A.data_ptr(), A[0].numel(), lda, int(a_mn),
           B.data_ptr(), B[0].numel(), ldb, int(b_mn), int(presplit),
           None if bv is None else bv.data_ptr(), Cm.data_ptr(), M * N_, N_, engine)
    Ad = A.double().transpose(1, 2) if a_mn else A.double()
    Bd = B.double().transpose(1, 2) if b_mn else B.double()
    ref = Ad @ Bd.transpose(1, 2)
    if bias:
        ref = ref + bv.double()
    return Cm.double(), ref


def relerr(c, ref):
    return float((c - ref).abs().max() / ref.abs().max())


SHAPES = [
    (1, 128, 128, 32, False, False, True),
    (1, 256, 384, 768, False, False, True),
    (2, 300, 200, 100, False, False, True),     # ragged M, N, K
    (3, 128, 256, 64, False, True, True),       # MN-major B (dgrad)
    (2, 192, 160, 256, True, True, False),      # wgrad: both MN-major, B split in smem
    (1, 96, 24, 12, False, False, True),        # tiny K < BK
    (4, 512, 768, 3072, False, False, True),    # BERT MLP-out shape (K=f)
    (1, 64, 768, 4096, True, True, False),      # wgrad-like K = tokens
]


@pytest.mark.parametrize("shape", SHAPES)
def test_tc_matches_fp64(shape):
    G, M, N_, K, a_mn, b_mn, pre = shape
    c, ref = run(G, M, N_, K, a_mn, b_mn, pre, engine=0, bias=True)
    assert not torch.isnan(c).any()
    e = relerr(c, ref)
    # tf32x3 with fp32 tensor-core accumulation: ~1e-6 at K~100, ~1e-5 at K=4096
    assert e < 2e-5, e


@pytest.mark.parametrize("shape", SHAPES[:5])
def test_simt_reference_kernel(shape):
    G, M, N_, K, a_mn, b_mn, pre = shape
    c, ref = run(G, M, N_, K, a_mn, b_mn, False, engine=1)
    assert relerr(c, ref) < 5e-6


def test_split_is_effective():
    """single-pass tf32 sits at ~8e-4 (measured); the 3-pass split with a
    separate correction accumulator must be fp32-class (~6e-6 at K=2048)"""
    c, ref = run(1, 256, 256, 2048, False, False, True, engine=0)
    assert relerr(c, ref) < 1.2e-5


_TRUNC_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2601_09026_b200 import _native as N
torch.manual_seed(0)
M, Nn, K = 256, 256, 512
A = torch.randn(M, K).float().cuda()
B = torch.randn(Nn, K).float().cuda()
C = torch.empty(M, Nn, device="cuda")
N.call("mglp_test_gemm", 1, M, Nn, K, A.data_ptr(), 0, K, 0, B.data_ptr(), 0, K, 0, 0, None,
       C.data_ptr(), 0, Nn, 0)
np.save(sys.argv[2], C.cpu().numpy())
"""


def test_tf32_operand_truncation(tmp_path):
    """kind::tf32 reads fp32 operands truncated to tf32: feeding the raw tile
    as the hi part (default) is bitwise identical to writing the masked hi
    (MGLP_TF32_EXPLICIT_HI=1). The default converter relies on this."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "t.py"
    script.write_text(_TRUNC_SCRIPT)
    outs = []
    for explicit in ("0", "1"):
        out = tmp_path / f"c{explicit}.npy"
        env = dict(os.environ, MGLP_TF32_EXPLICIT_HI=explicit)
        subprocess.run([sys.executable, str(script), root, str(out)], check=True, env=env)
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])
