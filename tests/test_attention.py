"""Fused tcgen05 attention (attn_tc.cu) against an fp64 torch restatement of
the reference's attention / vjp_attention (blocks.cpp:142-236: per-head
scores * 1/sqrt(dh), -1e30 causal mask, stable softmax_rows, P.V, and the VJP
dS = P (dP - rowsum(dP P))), through the C-ABI test hook."""
import math

import pytest

torch = pytest.importorskip("torch")
from paper_2601_09026_b200 import _native as N  # noqa: E402

pytestmark = pytest.mark.gpu


def reference(Q, K, V, dO, B, H, sq, skv, dh, causal):
    Qd, Kd, Vd, dOd = (t.double() for t in (Q, K, V, dO))
    O = torch.zeros(B, sq, H * dh, dtype=torch.float64)
    P = torch.zeros(B, H, sq, skv, dtype=torch.float64)
    dQ = torch.zeros_like(Qd[..., :H * dh])
    dK = torch.zeros(B, skv, H * dh, dtype=torch.float64)
    dV = torch.zeros(B, skv, H * dh, dtype=torch.float64)
    sc = 1.0 / math.sqrt(dh)
    for b in range(B):
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            q, k, v, do = Qd[b, :, sl], Kd[b, :, sl], Vd[b, :, sl], dOd[b, :, sl]
            s = q @ k.T * sc
            if causal:
                s = s.masked_fill(torch.ones(sq, skv).triu(1).bool(), -1e30)
            p = torch.softmax(s, dim=-1)
            P[b, h] = p
            O[b, :, sl] = p @ v
            dp = do @ v.T
            ds = p * (dp - (dp * p).sum(-1, keepdim=True))
            dQ[b, :, sl] = ds @ k * sc
            dK[b, :, sl] = ds.T @ q * sc
            dV[b, :, sl] = p.T @ do
    return O, P, dQ, dK, dV


def head_split(x):
    """fp32 rows -> the head-split pre-split form the QKV GEMM epilogue writes
    (common.cuh st_hs4): per 64 columns, 64 fp16 hi then 64 fp16 lo' =
    fp16((x - hi) * 2^11), the same bytes per row"""
    sh = x.shape
    y = x.reshape(*sh[:-1], -1, 64)
    hi = y.half()
    lo = ((y - hi.float()) * 2048.0).half()
    return torch.cat([hi, lo], -1).contiguous().view(torch.float32).reshape(sh).contiguous()


def run(B, H, sq, skv, dh, causal, seed=0, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    d = H * dh
    ld = 3 * d  # the qkv row layout of a layer
    qkv_q = torch.randn(B, sq, ld, generator=g) * scale
    qkv_kv = torch.randn(B, skv, ld, generator=g) * scale
    Q = qkv_q[..., :d].contiguous()
    K = qkv_kv[..., d:2 * d].contiguous()
    V = qkv_kv[..., 2 * d:].contiguous()
    dO = torch.randn(B, sq, d, generator=g)
    # device buffers with row stride ld (heads interleaved in a token row)
    dq = qkv_q.clone().cuda()
    dkv = qkv_kv.clone().cuda()
    ddo = torch.zeros(B, sq, ld, device="cuda")
    ddo[..., :d] = dO.cuda()
    if int(causal) & 4:  # operands in the head-split pre-split form (AttnArgs::qkv_hs / do_hs)
        dq, dkv = head_split(dq), head_split(dkv)
        if (sq <= 128 and skv <= 128) or int(causal) & 8:  # else the long backward reads fp32 dO
            ddo = head_split(ddo)
    O = torch.full((B, sq, ld), float("nan"), device="cuda")
    ldp = (skv + 3) & ~3
    P = torch.full((B, H, sq, ldp), float("nan"), device="cuda")
    dQ = torch.full((B, sq, ld), float("nan"), device="cuda")
    dKV = torch.full((B, skv, ld), float("nan"), device="cuda")
    N.call("mglp_test_attention", B, H, sq, skv, dh, int(causal), dq.data_ptr(),
           dkv[..., d:].data_ptr(), dkv[..., 2 * d:].data_ptr(), ld, O.data_ptr(), P.data_ptr(),
           ddo.data_ptr(), dQ.data_ptr(), dKV[..., d:].data_ptr(), dKV[..., 2 * d:].data_ptr(), None)
    ref = reference(Q, K, V, dO, B, H, sq, skv, dh, int(causal) & 1)
    got = (O[..., :d].cpu(), P[..., :skv].cpu(), dQ[..., :d].cpu(), dKV[..., d:2 * d].cpu(),
           dKV[..., 2 * d:].cpu())
    return got, ref


def relerr(a, b):
    return float((a.double() - b).abs().max() / b.abs().max())


SHAPES = [  # B, H, sq, skv, dh, causal
    (2, 2, 32, 32, 32, False),     # BASELINE configs[0] head shape
    (2, 3, 128, 128, 64, False),   # BERT / MT head shape
    (2, 2, 128, 128, 64, True),    # causal self-attention
    (1, 2, 64, 128, 64, False),    # cross-attention, sq != skv
    (2, 1, 128, 40, 32, False),    # skv not a multiple of 16 / 32
    (1, 2, 8, 8, 64, True),        # minimal sequence
    (1, 1, 96, 24, 64, False),
]


LONG_SHAPES = [  # attn_long.cu: key/query blocks of 128, P recomputed in the backward
    (1, 2, 512, 512, 64, True),    # GPT-2-style causal decoder
    (2, 2, 197, 197, 64, False),   # ViT-B/16 (197 tokens)
    (1, 1, 256, 384, 64, False),   # cross-attention, sq != skv
    (1, 2, 300, 300, 32, True),    # ragged blocks, dh 32
]


@pytest.mark.parametrize("shape", SHAPES + LONG_SHAPES)
def test_fused_attention_matches_fp64(shape):
    B, H, sq, skv, dh, causal = shape
    got, ref = run(B, H, sq, skv, dh, causal)
    names = ["O", "P", "dQ", "dK", "dV"]
    long_form = sq > 128 or skv > 128
    for n, a, b in zip(names, got, ref):
        if long_form and n == "P":
            continue  # the long form stores row statistics, not P
        assert not torch.isnan(a).any(), n
        e = relerr(a, b)
        assert e < 2e-5, (n, e)


def test_long_form_row_statistics():
    """P slot of the long form: per query row (max of the scaled masked
    scores, 1 / sum exp(s - max)) -- what the backward recomputes P from"""
    B, H, s, dh = 1, 1, 256, 64
    got, _ = run(B, H, s, s, dh, True, seed=5)
    g = torch.Generator().manual_seed(5)
    d = H * dh
    qkv_q = torch.randn(B, s, 3 * d, generator=g)
    qkv_kv = torch.randn(B, s, 3 * d, generator=g)
    q = qkv_q[0, :, :d].double()
    k = qkv_kv[0, :, d:2 * d].double()
    sc = (q @ k.T) / math.sqrt(dh)
    sc = sc.masked_fill(torch.ones(s, s).triu(1).bool(), float("-inf"))
    m = sc.max(-1).values
    inv = 1.0 / torch.exp(sc - m[:, None]).sum(-1)
    st = got[1].reshape(-1)[: 2 * s].reshape(s, 2).double()
    assert float((st[:, 0] - m).abs().max()) < 1e-4
    assert float(((st[:, 1] - inv) / inv).abs().max()) < 1e-4


def test_causal_probabilities_are_exactly_zero_above_diagonal():
    got, _ = run(1, 2, 64, 64, 64, True, seed=4)
    P = got[1]
    mask = torch.ones(64, 64).triu(1).bool()
    assert (P[..., mask] == 0).all()


def test_range_flag_on_fp16_overflow():
    B, H, s, dh = 1, 1, 32, 32
    d = H * dh
    x = torch.randn(B, s, 3 * d, device="cuda")
    x[0, 3, 5] = 1e5  # a query value beyond the fp16 split range
    O = torch.zeros(B, s, 3 * d, device="cuda")
    P = torch.zeros(B, H, s, s, device="cuda")
    import ctypes as C
    flag = C.c_int(0)
    N.call("mglp_test_attention", B, H, s, s, dh, 0, x.data_ptr(), x[..., d:].data_ptr(),
           x[..., 2 * d:].data_ptr(), 3 * d, O.data_ptr(), P.data_ptr(), None, None, None, None,
           C.byref(flag))
    assert flag.value == 1


def test_unsupported_shape_is_a_validation_error():
    x = torch.zeros(1, 600, 192, device="cuda")
    with pytest.raises(N.ValidationError):
        N.call("mglp_test_attention", 1, 1, 600, 600, 64, 0, x.data_ptr(), x.data_ptr(),
               x.data_ptr(), 192, x.data_ptr(), x.data_ptr(), None, None, None, None, None)


@pytest.mark.parametrize("causal", [False, True])
def test_presplit_p_is_bitwise_the_fp32_p_path(causal):
    """s = 128: the engine keeps P as the forward's hi|lo' operand tiles
    (bulk-copied out and back in) instead of fp32 probabilities; the backward
    converts an fp32 P into exactly those tiles, so O, dQ, dK, dV must agree
    bit for bit"""
    a, ref = run(2, 3, 128, 128, 64, causal, seed=5)
    b, _ = run(2, 3, 128, 128, 64, int(causal) | 2, seed=5)
    for n, x, y in zip(["O", "dQ", "dK", "dV"], (a[0],) + a[2:], (b[0],) + b[2:]):
        assert torch.equal(x, y), n
    assert relerr(b[0], ref[0]) < 1e-5


@pytest.mark.parametrize("shape", [s for s in SHAPES if s[4] == 64])
def test_presplit_operands_are_bitwise_the_fp32_path(shape):
    """Q, K, V and dO arriving head-split pre-split (TMA'd straight into the
    operand tiles) give bit-identical O, P, dQ, dK, dV: the kernel's own
    conversion of fp32 operands builds exactly those tiles"""
    B, H, sq, skv, dh, causal = shape
    a, ref = run(B, H, sq, skv, dh, causal, seed=7)
    b, _ = run(B, H, sq, skv, dh, int(causal) | 4, seed=7)
    for n, x, y in zip(["O", "P", "dQ", "dK", "dV"], a, b):
        assert torch.equal(x, y), n
    assert relerr(b[0], ref[0]) < 2e-5


@pytest.mark.parametrize("shape", [(1, 2, 512, 512, 64, True), (2, 2, 197, 197, 64, False),
                                   (1, 1, 256, 384, 64, False), (1, 3, 320, 320, 64, True)])
def test_flash_forward_presplit(shape):
    """128 < s <= 512 with head-split pre-split Q, K, V (attn_flash.cu):
    single-pass online softmax with P~ in TMEM. O against fp64, and the row
    statistics through their invariant m - log(1/l) = logsumexp_j(s_j scale)
    (the reference max m may lag the true max: lazy rescaling)"""
    B, H, sq, skv, dh, causal = shape
    g = torch.Generator().manual_seed(11)
    d = H * dh
    qkv_q = torch.randn(B, sq, 3 * d, generator=g)
    qkv_kv = torch.randn(B, skv, 3 * d, generator=g)
    dq, dkv = head_split(qkv_q.clone().cuda()), head_split(qkv_kv.clone().cuda())
    O = torch.full((B, sq, 3 * d), float("nan"), device="cuda")
    ldp = (skv + 3) & ~3
    P = torch.full((B, H, sq, ldp), float("nan"), device="cuda")
    N.call("mglp_test_attention", B, H, sq, skv, dh, int(causal) | 4, dq.data_ptr(),
           dkv[..., d:].data_ptr(), dkv[..., 2 * d:].data_ptr(), 3 * d, O.data_ptr(), P.data_ptr(),
           None, None, None, None, None)
    Q, K, V = qkv_q[..., :d], qkv_kv[..., d:2 * d], qkv_kv[..., 2 * d:]
    ref_O, _, _, _, _ = reference(Q, K, V, torch.zeros(B, sq, d), B, H, sq, skv, dh, causal)
    assert relerr(O[..., :d].cpu(), ref_O) < 2e-5
    st = P.cpu().reshape(B, H, -1)[..., : 2 * sq].reshape(B, H, sq, 2).double()
    for b in range(B):
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            s = (Q[b, :, sl].double() @ K[b, :, sl].double().T) / math.sqrt(dh)
            if causal:
                s = s.masked_fill(torch.ones(sq, skv).triu(1).bool(), float("-inf"))
            lse = torch.logsumexp(s, -1)
            got = st[b, h, :, 0] - torch.log(st[b, h, :, 1])
            assert float((got - lse).abs().max()) < 1e-5


@pytest.mark.parametrize("shape", [s for s in LONG_SHAPES if s[4] == 64])
def test_flash_presplit_forward_backward_matches_fp64(shape):
    """128 < s <= 512 with pre-split Q, K, V: the single-pass forward
    (attn_flash.cu) and the long backward reading the pre-split tiles"""
    B, H, sq, skv, dh, causal = shape
    got, ref = run(B, H, sq, skv, dh, int(causal) | 4, seed=3)
    for n, a, b in zip(["O", "P", "dQ", "dK", "dV"], got, ref):
        if n == "P":
            continue
        assert not torch.isnan(a).any(), n
        assert relerr(a, b) < 2e-5, (n, relerr(a, b))


@pytest.mark.parametrize("shape", [s for s in LONG_SHAPES if s[4] == 64] +
                         [(8, 12, 512, 512, 64, True)])  # several problems per CTA
def test_flash_backward_matches_fp64(shape):
    """128 < s <= 512, everything pre-split: single-pass forward and the
    single-pass backward (t_q row dot, dK / dV per key block storing the dS
    tiles, dQ per query block) against fp64"""
    B, H, sq, skv, dh, causal = shape
    got, ref = run(B, H, sq, skv, dh, int(causal) | 4 | 8, seed=9)
    for n, a, b in zip(["O", "P", "dQ", "dK", "dV"], got, ref):
        if n == "P":
            continue
        assert not torch.isnan(a).any(), n
        assert relerr(a, b) < 2e-5, (n, relerr(a, b))
