"""Frozen dropout masks on the device (blocks.cpp:576-599):
masks regenerated from the reference's counter streams (bit-identical keep /
drop decisions), applied at the attention / cross-attention / MLP outputs and
in their VJPs, against the compiled reference LayerStack with the same
refresh_dropout(seed, batch_index, ...) -- Phi, Phi^T with gradients, the
layer-parallel engine and a training run."""
import numpy as np
import pytest

from oracle import ref as R
from paper_2601_09026_b200 import LayerParallelEngine, LayerStack, SolveConfig, StackConfig, State

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="reference oracle not built")]

CASES = [  # kind, n_enc, n_dec, buffers, (B, sx, sy)
    ("encoder", 6, 0, (0, 0), (2, 6, 0)),
    ("decoder_only", 0, 6, (1, 1), (2, 7, 0)),
    ("encoder_decoder", 3, 3, (0, 0), (2, 5, 4)),
]


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(float(np.abs(b).max()), 1e-300))


def pair(kind, n_enc, n_dec, buffers, dropout=0.25, seed=13):
    cfg = StackConfig(kind=kind, d=16, heads=2, ffn=32, n_enc=n_enc, n_dec=n_dec,
                      buffer_open=buffers[0], buffer_close=buffers[1], dropout=dropout)
    st = LayerStack(cfg, seed)
    rc = R.RefStackConfig(kind=kind, d=16, heads=2, ffn=32, dropout=dropout)
    rc.n_enc, rc.n_dec = n_enc, n_dec
    rc.buffer_open, rc.buffer_close = buffers
    ref = R.RefStack(rc, seed)
    return st, ref


def draw(n, seed, scale=1.0):
    return R.gaussian_fill(seed, 6, seed, n, scale)


@pytest.mark.parametrize("case", CASES)
def test_step_and_adjoint_step_with_masks(case):
    kind, n_enc, n_dec, buf, (b, sx, sy) = case
    st, ref = pair(kind, n_enc, n_dec, buf)
    st.refresh_dropout(21, 3, b, sx, sy)
    ref.refresh_dropout(21, 3, b, sx, sy)
    n = ref.state_size(b, sx, sy)
    z, lam = draw(n, 5, 0.5), draw(n, 6)
    sz = State.from_flat(z, b, sx, sy, 16)
    sl = State.from_flat(lam, b, sx, sy, 16)
    for layer in range(st.total_layers()):
        got = st.step(layer, 0.41, sz).flat()
        want = ref.step(layer, 0.41, z, b, sx, sy)
        assert rel(got, want) < 1e-5, (layer, rel(got, want))
        g = st.zero_grads()
        got = st.adjoint_step(layer, 0.41, sz, sl, g, 0.5).flat()
        rg = np.zeros(ref.num_params())
        want = ref.adjoint_step(layer, 0.41, z, lam, b, sx, sy, grads=rg, gscale=0.5)
        assert rel(got, want) < 1e-5, (layer, rel(got, want))
        assert rel(g, rg) < 1e-5, (layer, rel(g, rg))


def test_masks_change_the_map_and_clear_restores_it():
    st, ref = pair("encoder", 4, 0, (0, 0), dropout=0.5)
    b, sx = 2, 8
    n = ref.state_size(b, sx, 0)
    z = State.from_flat(draw(n, 9, 0.5), b, sx, 0, 16)
    plain = st.step(1, 1.0, z).flat()
    st.refresh_dropout(1, 0, b, sx, 0)
    masked = st.step(1, 1.0, z).flat()
    st.refresh_dropout(1, 1, b, sx, 0)
    other = st.step(1, 1.0, z).flat()
    st.clear_dropout()
    again = st.step(1, 1.0, z).flat()
    assert rel(masked, plain) > 1e-3 and rel(other, masked) > 1e-3
    assert np.array_equal(again, plain)


@pytest.mark.parametrize("case", CASES)
def test_engine_with_masks_matches_reference(case):
    kind, n_enc, n_dec, buf, (b, sx, sy) = case
    st, ref = pair(kind, n_enc, n_dec, buf)
    st.refresh_dropout(4, 9, b, sx, sy)
    ref.refresh_dropout(4, 9, b, sx, sy)
    n = ref.state_size(b, sx, sy)
    z0, lam = draw(n, 2, 0.5), draw(n, 3)
    interior = st.interior_end() - st.interior_begin()
    cf = 3 if interior % 3 == 0 else 2
    eng = LayerParallelEngine(st, SolveConfig(coarsen=cf, levels=2, fwd_iters=2, bwd_iters=2,
                                              warm_start=False))
    reng = R.RefEngine(ref, coarsen=cf, levels=2, fwd_iters=2, bwd_iters=2, warm_start=False)
    fo = eng.forward(State.from_flat(z0, b, sx, sy, 16))
    rtraj, rft, _ = reng.forward(z0, b, sx, sy)
    assert rel(np.stack([s.flat() for s in fo.traj]), rtraj) < 1e-4
    assert rel(fo.phase.trace, rft) < 1e-4
    g = st.zero_grads()
    bo = eng.backward(fo.traj, State.from_flat(lam, b, sx, sy, 16), g)
    rg = np.zeros(ref.num_params())
    rl0, rbt, _ = reng.backward(rtraj, lam, b, sx, sy, grads=rg)
    assert rel(bo.lambda0.flat(), rl0) < 1e-4
    assert rel(bo.phase.trace, rbt) < 1e-4
    assert rel(g, rg) < 1e-4


def test_training_with_dropout_tracks_reference():
    """run_training refreshes the masks per batch (training.cpp:209-210) and
    evaluates on the exact map (training.cpp:296-300)"""
    from paper_2601_09026_b200 import training as T
    stack = StackConfig(kind="encoder", d=32, heads=2, ffn=64, n_enc=8, dropout=0.2)
    tk = T.TaskSpec(kind="copy_sequence", vocab=16, seq_len=8, train_size=16, val_size=8, seed=1)
    mc = T.ModelConfig(stack=stack, vocab=16, max_seq=8)
    tc = T.TrainConfig(mode="layer_parallel",
                       solve=SolveConfig(coarsen=2, levels=2, fwd_iters=2, bwd_iters=1),
                       batch_size=4, epochs=1, seed=7, val_every=2)
    ref = R.run_training(tk, mc, tc)
    res = T.run_training(tk, mc, tc)
    rl = [float(line.split(",")[1]) for line in ref["csv"].strip().splitlines()[1:]]
    assert len(res.rows) == len(rl)
    for d, r in zip(res.rows, rl):
        assert abs(d.loss - r) <= 1e-4 * abs(r), (d.batch, d.loss, r)
