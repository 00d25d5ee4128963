"""the training edge around the engine -- synthetic
batches, embedding, head / cross-entropy, embedding backward, the optimizer
and the MGLP v1 checkpoint -- against the compiled reference
(oracle/_ref: tasks.cpp, model.cpp, optimizer.cpp, checkpoint.cpp,
training.cpp run unmodified).

CPU tests pin the host-side pieces (config echo, metrics CSV, checkpoint
parser) on reference outputs; GPU tests compare the device Trainer with
reference run_training: tokens bit-exact, initial parameters bit-exact,
losses / gradients within the north-star 1e-4 relative tolerance.
"""
import numpy as np
import pytest

from oracle import ref as R
from paper_2601_09026_b200.engine import SolveConfig, StackConfig
from paper_2601_09026_b200.controller import IndicatorConfig
from paper_2601_09026_b200 import training as T

pytestmark = pytest.mark.skipif(not R.available(), reason="reference oracle not built")


def small(kind="encoder", task="copy_sequence", mode="layer_parallel", epochs=1, train=16,
          **kw):
    n_enc, n_dec = {"encoder": (8, 0), "decoder_only": (0, 8), "encoder_decoder": (4, 4)}[kind]
    stack = StackConfig(kind=kind, d=32, heads=2, ffn=64, n_enc=n_enc, n_dec=n_dec)
    tk = T.TaskSpec(kind=task, vocab=16, seq_len=8, train_size=train, val_size=8, seed=1)
    mc = T.ModelConfig(stack=stack, vocab=16, max_seq=8)
    tc = T.TrainConfig(mode=mode, solve=SolveConfig(coarsen=2, levels=2, fwd_iters=2, bwd_iters=1),
                       batch_size=4, epochs=epochs, seed=7, val_every=2, **kw)
    return tk, mc, tc


def parse_csv(csv):
    rows = []
    for line in csv.strip().splitlines()[1:]:
        f = [x.strip() for x in line.split(",")]
        rows.append(T.MetricsRow(int(f[0]), float(f[1]), float(f[2]), f[3], int(f[4]), int(f[5]),
                                 float(f[6]), float(f[7])))
    return rows


# ---- host side (CPU) ----------------------------------------------------------------
@pytest.mark.parametrize("args", [("encoder", "copy_sequence"),
                                  ("decoder_only", "token_classification"),
                                  ("encoder_decoder", "tiny_translation")])
def test_config_echo_matches_reference(args):
    tk, mc, tc = small(*args)
    tc.opt.lr = 3e-4
    tc.opt.weight_decay = 0.1
    assert T.config_echo(tk, mc, tc) == R.config_echo(tk, mc, tc)


def test_checkpoint_parser_and_csv_on_reference_run():
    tk, mc, tc = small()
    out = R.run_training(tk, mc, tc)
    ck = T.parse_checkpoint(out["final_state"])
    assert ck["version"] == 1 and ck["batch"] == 4
    assert ck["config_echo"] == T.config_echo(tk, mc, tc)
    _, shapes = R.model_params(mc, tc.seed)
    assert [t.shape for t in ck["params"]] == list(shapes)
    assert ck["has_optimizer"] and ck["steps"] == 4
    assert len(ck["m"]) == len(shapes) == len(ck["v"])
    assert T.metrics_csv(parse_csv(out["csv"])) == out["csv"]


# ---- device (GPU) -------------------------------------------------------------------
gpu = pytest.mark.gpu


@gpu
@pytest.mark.parametrize("task", ["copy_sequence", "token_classification", "tiny_translation"])
def test_device_batches_bit_exact(task):
    kind = "encoder_decoder" if task == "tiny_translation" else "encoder"
    tk, mc, tc = small(kind, task)
    dev = T.DeviceTrainer(tk, mc, tc)
    for split, start in [(0, 0), (0, 12), (1, 4), (0, 1 << 40)]:
        src, tin, tout = dev.read_batch(split, start)
        rs, rti, rto = R.make_batch(tk, split, start, tc.batch_size)
        assert np.array_equal(src, rs) and np.array_equal(tout, rto)
        if rti is not None:
            assert np.array_equal(tin, rti)


@gpu
@pytest.mark.parametrize("kind", ["encoder", "encoder_decoder"])
def test_device_model_init_bit_exact(kind):
    tk, mc, tc = small(kind, "tiny_translation" if kind == "encoder_decoder" else "copy_sequence")
    dev = T.DeviceTrainer(tk, mc, tc)
    flat, _ = R.model_params(mc, tc.seed)
    assert np.array_equal(dev.params(), flat)


def relerr(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


@gpu
@pytest.mark.parametrize("args", [("encoder", "copy_sequence", "layer_parallel"),
                                  ("encoder", "token_classification", "serial"),
                                  ("decoder_only", "copy_sequence", "layer_parallel"),
                                  ("encoder_decoder", "tiny_translation", "layer_parallel")])
def test_one_update_matches_reference(args):
    """loss of batch 0 and every gradient (through Adam's first moment,
    m = (1 - beta1) g) after one AdamW step"""
    kind, task, mode = args
    tk, mc, tc = small(kind, task, mode, train=4)
    ref = R.run_training(tk, mc, tc)
    rrows = parse_csv(ref["csv"])
    rck = T.parse_checkpoint(ref["final_state"])
    res = T.run_training(tk, mc, tc)
    assert len(res.rows) == 1
    assert abs(res.rows[0].loss - rrows[0].loss) <= 1e-5 * abs(rrows[0].loss)
    dck = T.parse_checkpoint(res.final_state)
    assert dck["steps"] == rck["steps"] == 1
    # per tensor, relative to its own scale -- or to 1e-3 of the largest
    # gradient for tensors whose exact gradient is zero (the attention key
    # bias: softmax is shift invariant, both sides hold rounding noise)
    gmax = max(np.abs(rm).max() for rm in rck["m"])
    for i, (dm, rm) in enumerate(zip(dck["m"], rck["m"])):
        den = max(np.abs(rm).max(), 1e-3 * gmax)
        err = float(np.abs(dm - rm).max() / den)
        assert err < 1e-4, (i, err)


@gpu
@pytest.mark.parametrize("mode", ["layer_parallel", "serial"])
def test_training_run_tracks_reference(mode):
    """8 AdamW steps (2 epochs): per-batch losses, validation accuracy and the
    final parameters stay with the reference's run_training"""
    tk, mc, tc = small(mode=mode, epochs=2)
    ref = R.run_training(tk, mc, tc)
    res = T.run_training(tk, mc, tc)
    rrows = parse_csv(ref["csv"])
    assert [r.batch for r in res.rows] == [r.batch for r in rrows]
    assert [r.mode for r in res.rows] == [r.mode for r in rrows]
    for d, r in zip(res.rows, rrows):
        assert abs(d.loss - r.loss) <= 1e-4 * abs(r.loss), (d.batch, d.loss, r.loss)
        assert abs(d.val_metric - r.val_metric) <= 2.0 / 32 + 1e-12
        assert (d.fwd_iters, d.bwd_iters) == (r.fwd_iters, r.bwd_iters)
    dp = np.concatenate([t.ravel() for t in T.parse_checkpoint(res.final_state)["params"]])
    rp = np.concatenate([t.ravel() for t in T.parse_checkpoint(ref["final_state"])["params"]])
    assert relerr(dp, rp) < 1e-4


@gpu
def test_checkpoint_roundtrip_is_byte_identical():
    """a reference checkpoint loaded into the device trainer and saved again
    reproduces the reference bytes (f64 masters, same container)"""
    tk, mc, tc = small()
    ref = R.run_training(tk, mc, tc)
    dev = T.DeviceTrainer(tk, mc, tc)
    batch, echo, has = dev.load_checkpoint(ref["final_state"])
    assert (batch, echo, has) == (4, T.config_echo(tk, mc, tc), True)
    assert dev.save_checkpoint(batch, echo) == ref["final_state"]


@gpu
def test_resume_rejects_foreign_checkpoint():
    tk, mc, tc = small()
    ref = R.run_training(tk, mc, tc)
    tc2 = small()[2]
    tc2.seed = 8
    tr = T.Trainer(tk, mc, tc2)
    with pytest.raises(T.ValidationError):
        tr.resume_serial(ref["final_state"])


@gpu
def test_switching_replay_is_bitwise():
    """training.cpp:362-396 on the device: the serial tail replayed from the
    handover checkpoint reproduces every post-switch loss and the final state
    bit for bit"""
    tk, mc, tc = small(mode="switching", epochs=2, manual_switch_batch=3,
                       indicator=IndicatorConfig(probe_period=2))
    out = T.switching_replay(tk, mc, tc)
    assert out.switched and out.switch_batch == 3
    assert out.compared_batches == 5
    assert out.losses_match and out.state_matches


@gpu
def test_warm_start_survives_evaluation():
    """evaluation (a serial sweep) must not become the next batch's
    warm start. A 16-layer stack with c_f=4 and ONE forward / backward cycle
    per batch, so the initial guess changes every inexact solve, evaluated
    after every batch (val_every=1): losses, validation accuracy and final
    parameters track the reference's run_training, whose evaluation never
    touches the engine's solver states (training.cpp:280-293)."""
    stack = StackConfig(kind="encoder", d=32, heads=2, ffn=64, n_enc=16)
    tk = T.TaskSpec(kind="copy_sequence", vocab=16, seq_len=8, train_size=16, val_size=8, seed=1)
    mc = T.ModelConfig(stack=stack, vocab=16, max_seq=8)
    tc = T.TrainConfig(mode="layer_parallel",
                       solve=SolveConfig(coarsen=4, levels=2, fwd_iters=1, bwd_iters=1),
                       batch_size=4, epochs=2, seed=7, val_every=1)
    ref = R.run_training(tk, mc, tc)
    res = T.run_training(tk, mc, tc)
    rrows = parse_csv(ref["csv"])
    assert len(res.rows) == len(rrows) == 8
    for d, r in zip(res.rows, rrows):
        assert abs(d.loss - r.loss) <= 1e-4 * abs(r.loss), (d.batch, d.loss, r.loss)
    dp = np.concatenate([t.ravel() for t in T.parse_checkpoint(res.final_state)["params"]])
    rp = np.concatenate([t.ravel() for t in T.parse_checkpoint(ref["final_state"])["params"]])
    assert relerr(dp, rp) < 1e-4


@gpu
def test_one_update_at_4096_tokens(mode="layer_parallel"):
    """a batch of 32 x 128 = 4096 tokens, so the mean-token
    cross entropy puts lambda_N at O(1e-5) (model.cpp:213-248) -- the regime
    the fp16 split would lose to subnormals without the adjoint's 2^k scaling
    (the parameter gradients sum 4096 such rows, so they are O(0.1) again).
    Loss and every gradient (Adam's first moment) against run_training."""
    stack = StackConfig(kind="encoder", d=32, heads=2, ffn=64, n_enc=8)
    tk = T.TaskSpec(kind="copy_sequence", vocab=16, seq_len=128, train_size=32, val_size=32,
                    seed=1)
    mc = T.ModelConfig(stack=stack, vocab=16, max_seq=128)
    tc = T.TrainConfig(mode=mode, solve=SolveConfig(coarsen=2, levels=2, fwd_iters=2, bwd_iters=1),
                       batch_size=32, epochs=1, seed=7, val_every=2)
    ref = R.run_training(tk, mc, tc)
    rrows = parse_csv(ref["csv"])
    res = T.run_training(tk, mc, tc)
    assert len(res.rows) == 1
    assert abs(res.rows[0].loss - rrows[0].loss) <= 1e-5 * abs(rrows[0].loss)
    rck = T.parse_checkpoint(ref["final_state"])
    dck = T.parse_checkpoint(res.final_state)
    gmax = max(np.abs(rm).max() for rm in rck["m"])
    for i, (dm, rm) in enumerate(zip(dck["m"], rck["m"])):
        den = max(np.abs(rm).max(), 1e-3 * gmax)
        err = float(np.abs(dm - rm).max() / den)
        assert err < 1e-4, (i, err)
