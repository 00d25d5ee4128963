"""TEST INFRASTRUCTURE: full-depth parity summaries shared by the fixture
generator (tests/golden/make_deep.py, run in the build container against the
float64 numpy oracle pinned to the compiled reference) and the GPU parity
tests (tests/test_deep_parity.py).

At BASELINE's real depths a full trajectory / gradient dump is GBs, so each
output is summarised by size-independent statistics that still see every
entry:

* states: per time point the L2 norm, the values at 2048 fixed indices, and
  the whole final state;
* gradients: per (layer, component) the L2 norm, the max |g|, 128 values at
  fixed indices, and K=8 Rademacher sketches  s_k = sum_i r_k(i) g(i)  with
  r_k(i) = +-1 from a splitmix64 hash of (k, i). For an error E = g_dev - g_ref
  the sketch difference  s_k(dev) - s_k(ref) = <r_k, E>  has E[<r_k,E>^2] =
  ||E||_F^2, so the RMS of the K sketch differences estimates the Frobenius
  error of the WHOLE tensor (every entry contributes), and is compared with
  ||g_ref||_F.

Configs follow BASELINE.json configs[1..4] at their own depth, width, heads,
sequence length, c_f and number of levels, at batch 1 (B=1: the per-sample
computation is identical for every batch row, blocks.cpp:476-486).
Inputs: parameters LayerStack(cfg, seed 7) (blocks.cpp:432-449), z0 =
0.5*rng::gaussian(7, kTestOnly, 7, i), lambda_N = rng::gaussian(8, kTestOnly,
8, i) over the whole state -- exactly bench.py's generators.
"""
from __future__ import annotations

import numpy as np

K_TEST = 6
N_STATE_IDX = 2048
N_GRAD_IDX = 128
N_SKETCH = 8

DEEP = {
    # BASELINE configs[1]: BERT-base-style encoder, 2-level c_f=4
    "bert_deep": dict(kind="encoder", n_enc=64, n_dec=0, d=768, heads=12, ffn=3072, sx=128, sy=0,
                      B=1, cf=4, levels=2, fwd_iters=1, bwd_iters=1),
    # configs[2]: GPT-2-small-style causal decoder, 3-level c_f=4, s=512
    "gpt_deep": dict(kind="decoder_only", n_enc=0, n_dec=128, d=768, heads=12, ffn=3072, sx=512,
                     sy=0, B=1, cf=4, levels=3, fwd_iters=1, bwd_iters=1),
    # configs[3]: ViT-B/16-style encoder, 197 tokens, 2-level c_f=8
    "vit_deep": dict(kind="encoder", n_enc=64, n_dec=0, d=768, heads=12, ffn=3072, sx=197, sy=0,
                     B=1, cf=8, levels=2, fwd_iters=1, bwd_iters=1),
    # configs[4]: encoder-decoder 32+32, d=512, one stacked solve (Eq. 3)
    "mt_deep": dict(kind="encoder_decoder", n_enc=32, n_dec=32, d=512, heads=8, ffn=2048, sx=128,
                    sy=128, B=1, cf=4, levels=2, fwd_iters=1, bwd_iters=1),
}

# the bench's own workload (configs[1] at batch 32): first-cycle traces,
# lambda_0 and the final state
BENCH_BERT = dict(DEEP["bert_deep"], B=32)


def state_len(c):
    return c["B"] * (c["sx"] + c["sy"]) * c["d"]


def index_set(n, k, seed):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(n, k), replace=False)).astype(np.int64)


def _splitmix(x):
    x = (x + np.uint64(0x9E3779B97F4A7C15))
    z = x.copy()
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


_SIGNS = {}


def signs(n):
    """[N_SKETCH, n] float64 +-1 matrix, deterministic (integer hash)."""
    cached = _SIGNS.get("m")
    if cached is None or cached.shape[1] < n:
        i = np.arange(n, dtype=np.uint64)
        rows = []
        with np.errstate(over="ignore"):
            for k in range(N_SKETCH):
                h = _splitmix(i ^ (np.uint64(k + 1) << np.uint64(40)))
                rows.append(1.0 - 2.0 * (h >> np.uint64(63)).astype(np.float64))
        cached = np.stack(rows)
        _SIGNS["m"] = cached
    return cached[:, :n]


def components(kind, n_enc, d, ffn, layer):
    """(name, size) in visit_params order (blocks.cpp:627-646)."""
    dec = kind == "encoder_decoder" and layer >= n_enc

    def lin(p, o, i):
        return [(p + ".w", o * i), (p + ".b", o)]

    def ln(p):
        return [(p + ".gain", d), (p + ".bias", d)]

    def attn(p):
        return sum((lin(f"{p}.{k}", d, d) for k in "qkvo"), [])

    if not dec:
        return ln("ln1") + attn("attn") + ln("ln2") + lin("mlp.in", ffn, d) + lin("mlp.out", d, ffn)
    return (ln("ln1") + attn("self") + ln("ln3") + attn("cross") + ln("ln2")
            + lin("mlp.in", ffn, d) + lin("mlp.out", d, ffn))


def grad_summary(c, flat):
    """Per (layer, component): norm, maxabs, sketches, sampled values."""
    total = c["n_enc"] + c["n_dec"]
    norms, maxs, sk, samp = [], [], [], []
    o = 0
    for layer in range(total):
        for j, (name, n) in enumerate(components(c["kind"], c["n_enc"], c["d"], c["ffn"], layer)):
            g = np.asarray(flat[o:o + n], np.float64)
            o += n
            norms.append(float(np.sqrt(np.dot(g, g))))
            maxs.append(float(np.abs(g).max()))
            sk.append(signs(n) @ g)
            samp.append(g[index_set(n, N_GRAD_IDX, 1000 + n)])
    assert o == flat.size, (o, flat.size)
    return dict(g_norm=np.array(norms), g_max=np.array(maxs), g_sketch=np.stack(sk),
                g_samp=np.concatenate(samp))


def grad_errors(c, dev_flat, ref):
    """(max sketch-estimated relative Frobenius error, max sampled-entry error
    relative to the tensor's max |g|, max relative norm error), over all
    (layer, component) tensors."""
    d = grad_summary(c, dev_flat)
    den = np.maximum(ref["g_norm"], 1e-300)
    est = np.sqrt(np.mean((d["g_sketch"] - ref["g_sketch"]) ** 2, axis=1)) / den
    norm_err = np.abs(d["g_norm"] - ref["g_norm"]) / den
    # sampled entries against each tensor's max |g|
    total = c["n_enc"] + c["n_dec"]
    mx = []
    for layer in range(total):
        for _, n in components(c["kind"], c["n_enc"], c["d"], c["ffn"], layer):
            mx.append(np.full(min(n, N_GRAD_IDX), 1.0))
    reps = np.concatenate(mx)
    cnt = [int(r.size) for r in mx]
    scale = np.repeat(np.maximum(ref["g_max"], 1e-300), cnt)
    samp_err = np.abs(d["g_samp"] - ref["g_samp"]) / scale * reps
    return float(est.max()), float(samp_err.max()), float(norm_err.max())


def state_summary(c, traj):
    """traj: sequence of flat states (total+1)."""
    n = state_len(c)
    idx = index_set(n, N_STATE_IDX, 77)
    norms = np.array([float(np.linalg.norm(np.asarray(t, np.float64)[:n])) for t in traj])
    samp = np.stack([np.asarray(t, np.float64)[:n][idx] for t in traj])
    return dict(s_norm=norms, s_samp=samp, s_idx=idx)
