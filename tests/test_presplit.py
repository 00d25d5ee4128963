"""Pre-split operand paths against the compiled reference: with d, ffn and
the head width multiples of 32 every forward and dgrad GEMM reads its A
operand pre-split (LayerNorm, attention O / dQKV, GELU and GELU' epilogues,
LayerNorm VJP, the upstream pack), for all three stack kinds including
cross-attention, with ffn < 3d (the dQKV rows are the widest pre-split
buffer). The small golden stacks (d = 16) never take these paths."""
import numpy as np
import pytest

from oracle import ref as R
from paper_2601_09026_b200 import LayerParallelEngine, LayerStack, SolveConfig, StackConfig, State

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="reference oracle not built")]

D, H, F = 64, 2, 96
CASES = [  # kind, n_enc, n_dec, (B, sx, sy), causal buffers
    ("encoder", 6, 0, (2, 16, 0), (0, 0)),
    ("decoder_only", 0, 6, (2, 24, 0), (1, 1)),
    ("encoder_decoder", 3, 3, (2, 16, 8), (0, 0)),
    # s = 128: the fused attention keeps P pre-split (bulk-copied out by the
    # forward, back in by the backward) inside the engine's solve
    ("encoder", 4, 0, (1, 128, 0), (0, 0)),
    ("decoder_only", 0, 4, (1, 128, 0), (0, 0)),
    # s = 256: the streamed long attention; its dK/dV kernel stores the dS
    # tiles pre-split and the dQ kernel reads them back
    ("encoder", 4, 0, (1, 256, 0), (0, 0)),
    ("decoder_only", 0, 4, (1, 256, 0), (0, 0)),
    ("encoder", 4, 0, (2, 200, 0), (0, 0)),  # ragged blocks (padded dS tiles)
    # long self- and cross-attention (sq = 192 queries over 256 encoder keys)
    ("encoder_decoder", 2, 2, (1, 256, 192), (0, 0)),
]


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(float(np.abs(b).max()), 1e-300))


@pytest.mark.parametrize("case", CASES)
def test_engine_with_presplit_operands_matches_reference(case):
    kind, n_enc, n_dec, (b, sx, sy), buf = case
    cfg = StackConfig(kind=kind, d=D, heads=H, ffn=F, n_enc=n_enc, n_dec=n_dec,
                      buffer_open=buf[0], buffer_close=buf[1])
    st = LayerStack(cfg, 11)
    rc = R.RefStackConfig(kind=kind, d=D, heads=H, ffn=F)
    rc.n_enc, rc.n_dec = n_enc, n_dec
    rc.buffer_open, rc.buffer_close = buf
    ref = R.RefStack(rc, 11)
    n = ref.state_size(b, sx, sy)
    z0 = R.gaussian_fill(2, 6, 2, n, 0.5)
    lam = R.gaussian_fill(3, 6, 3, n, 1.0)
    interior = st.interior_end() - st.interior_begin()
    cf = 3 if interior % 3 == 0 else 2
    eng = LayerParallelEngine(st, SolveConfig(coarsen=cf, levels=2, fwd_iters=2, bwd_iters=2,
                                              warm_start=False))
    reng = R.RefEngine(ref, coarsen=cf, levels=2, fwd_iters=2, bwd_iters=2, warm_start=False)
    fo = eng.forward(State.from_flat(z0, b, sx, sy, D))
    rtraj, rft, _ = reng.forward(z0, b, sx, sy)
    assert rel(np.stack([s.flat() for s in fo.traj]), rtraj) < 1e-4
    assert rel(fo.phase.trace, rft) < 1e-4
    g = st.zero_grads()
    bo = eng.backward(fo.traj, State.from_flat(lam, b, sx, sy, D), g)
    rg = np.zeros(ref.num_params())
    rl0, rbt, _ = reng.backward(rtraj, lam, b, sx, sy, grads=rg)
    assert rel(bo.lambda0.flat(), rl0) < 1e-4
    assert rel(bo.phase.trace, rbt) < 1e-4
    assert rel(g, rg) < 1e-4


@pytest.mark.parametrize("sx", [16, 256])
def test_presplit_operands_with_dropout_masks(sx):
    """dropout sites on the pre-split paths: the masked O-projection / MLP-out
    epilogues, the masked LayerNorm VJP output written pre-split (da1) and
    the masked upstream copy packed for the GELU' dgrad (s = 256: with the
    long attention and its stored dS tiles)"""
    b = 2 if sx == 16 else 1
    cfg = StackConfig(kind="encoder", d=D, heads=H, ffn=F, n_enc=4, dropout=0.25)
    st = LayerStack(cfg, 5)
    rc = R.RefStackConfig(kind="encoder", d=D, heads=H, ffn=F, dropout=0.25)
    rc.n_enc, rc.n_dec = 4, 0
    ref = R.RefStack(rc, 5)
    st.refresh_dropout(3, 7, b, sx, 0)
    ref.refresh_dropout(3, 7, b, sx, 0)
    n = ref.state_size(b, sx, 0)
    z0 = R.gaussian_fill(4, 6, 4, n, 0.5)
    lam = R.gaussian_fill(5, 6, 5, n, 1.0)
    eng = LayerParallelEngine(st, SolveConfig(coarsen=2, levels=2, fwd_iters=2, bwd_iters=2,
                                              warm_start=False))
    reng = R.RefEngine(ref, coarsen=2, levels=2, fwd_iters=2, bwd_iters=2, warm_start=False)
    fo = eng.forward(State.from_flat(z0, b, sx, 0, D))
    rtraj, rft, _ = reng.forward(z0, b, sx, 0)
    assert rel(np.stack([s.flat() for s in fo.traj]), rtraj) < 1e-4
    assert rel(fo.phase.trace, rft) < 1e-4
    g = st.zero_grads()
    bo = eng.backward(fo.traj, State.from_flat(lam, b, sx, 0, D), g)
    rg = np.zeros(ref.num_params())
    rl0, rbt, _ = reng.backward(rtraj, lam, b, sx, 0, grads=rg)
    assert rel(bo.lambda0.flat(), rl0) < 1e-4
    assert rel(bo.phase.trace, rbt) < 1e-4
    assert rel(g, rg) < 1e-4


def test_training_on_presplit_sizes_tracks_reference():
    """the device training step (trainer.cu: head, loss, adjoint, optimizer)
    with every GEMM operand pre-split, against the reference's run_training"""
    from paper_2601_09026_b200 import training as T
    stack = StackConfig(kind="encoder", d=D, heads=H, ffn=F, n_enc=4)
    tk = T.TaskSpec(kind="copy_sequence", vocab=16, seq_len=16, train_size=16, val_size=8, seed=2)
    mc = T.ModelConfig(stack=stack, vocab=16, max_seq=16)
    tc = T.TrainConfig(mode="layer_parallel",
                       solve=SolveConfig(coarsen=2, levels=2, fwd_iters=2, bwd_iters=1),
                       batch_size=4, epochs=1, seed=3, val_every=2)
    ref = R.run_training(tk, mc, tc)
    res = T.run_training(tk, mc, tc)
    rl = [float(line.split(",")[1]) for line in ref["csv"].strip().splitlines()[1:]]
    assert len(res.rows) == len(rl)
    for d, r in zip(res.rows, rl):
        assert abs(d.loss - r) <= 1e-4 * abs(r), (d.batch, d.loss, r)
