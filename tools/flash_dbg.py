"""Diagnostics: per-shape errors of the single-pass attention (fwd stats, dQ, dK, dV)."""
import math
import sys

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import torch  # noqa: E402
from test_attention import relerr, run  # noqa: E402

for shape in [(8, 12, 512, 512, 64, True), (4, 12, 512, 512, 64, True), (8, 12, 256, 256, 64, False)]:
    B, H, sq, skv, dh, causal = shape
    got, ref = run(B, H, sq, skv, dh, int(causal) | 4 | 8, seed=9)
    errs = {n: relerr(a, b) for n, a, b in zip(["O", "P", "dQ", "dK", "dV"], got, ref) if n != "P"}
    # forward statistics: m - log(1/l) = logsumexp
    g = torch.Generator().manual_seed(9)
    d = H * dh
    qkv_q = torch.randn(B, sq, 3 * d, generator=g)
    qkv_kv = torch.randn(B, skv, 3 * d, generator=g)
    st = got[1].reshape(B, H, -1)[..., : 2 * sq].reshape(B, H, sq, 2).double()
    bad = []
    for b in range(B):
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            s = (qkv_q[b, :, sl].double() @ qkv_kv[b, :, d + h * dh:d + (h + 1) * dh].double().T) / math.sqrt(dh)
            if causal:
                s = s.masked_fill(torch.ones(sq, skv).triu(1).bool(), float("-inf"))
            e = float((st[b, h, :, 0] - torch.log(st[b, h, :, 1]) - torch.logsumexp(s, -1)).abs().max())
            if e > 1e-4:
                bad.append((b, h, e))
    dq, rdq = got[2], ref[2]
    badq = []
    for b in range(B):
        for h in range(H):
            e = float((dq[b, :, h * dh:(h + 1) * dh].double() - rdq[b, :, h * dh:(h + 1) * dh]).abs().max() / rdq.abs().max())
            if e > 1e-5:
                badq.append((b, h, f"{e:.1e}"))
    print(shape, {k: f"{v:.1e}" for k, v in errs.items()}, "bad stats", bad[:6], len(bad), "bad dQ heads", badq[:8], len(badq))
