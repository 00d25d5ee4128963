"""Lipschitz probe and buffer-layer selection: the
device probe against the compiled reference's estimate_lipschitz
(lipschitz.cpp:53-149), and the host rules against the reference's own test
cases (test_lipschitz.cpp:144-300) and the compiled reference."""
import numpy as np
import pytest

from oracle import ref as R
from paper_2601_09026_b200 import lipschitz as L
from paper_2601_09026_b200._native import ContractViolation, ValidationError

needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def synth(vals):
    return [L.LipschitzEstimate(layer=i, estimate=v) for i, v in enumerate(vals)]


# ---- host rules (no GPU) ------------------------------------------------------

def test_buffer_selection_known_answers():
    """test_lipschitz.cpp:144-184"""
    vals = [0.3] * 20
    vals[0] = vals[1] = vals[18] = vals[19] = 3.0
    plan = L.select_buffer_layers(synth(vals), 2, 2)
    assert plan.buffered == [0, 1, 18, 19]
    assert not plan.interior_spike and plan.warning == ""
    vals = [0.3] * 20
    vals[0] = vals[19] = 1.0
    vals[9] = 5.0
    plan = L.select_buffer_layers(synth(vals), 1, 1)
    assert plan.interior_spike and plan.warning
    plan = L.select_buffer_layers(synth([1.0] * 8), 0, 0)
    assert plan.buffered == [] and not plan.interior_spike
    with pytest.raises(ValidationError):
        L.select_buffer_layers(synth([1.0] * 4), 2, 2)


def test_buffer_recommendation_known_answers():
    """test_lipschitz.cpp:282-300"""
    r = L.recommend_buffers([1.2] * 8)
    assert (r.k_open, r.k_close) == (0, 0)
    r = L.recommend_buffers([5.0, 3.0, 1.1, 1.2, 1.1, 1.0, 2.5, 4.0])
    assert (r.k_open, r.k_close) == (2, 2)
    r = L.recommend_buffers([3.0, 1.1, 9.0, 1.1, 1.1, 1.0])
    assert (r.k_open, r.k_close) == (1, 0)
    with pytest.raises(ValidationError):
        L.recommend_buffers([1.0, 2.0], amp_threshold=1.0)


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_host_rules_match_reference(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 24))
    amps = 1.0 + rng.exponential(0.8, n)
    thr = 1.5 + rng.random()
    assert (lambda r: (r.k_open, r.k_close))(L.recommend_buffers(list(amps), amp_threshold=thr)) \
        == R.lipschitz_recommend(amps, thr)
    est = rng.exponential(1.0, n)
    ko = int(rng.integers(0, max(1, (n - 1) // 2)))
    kc = int(rng.integers(0, max(1, n - 1 - ko)))
    plan = L.select_buffer_layers(synth(list(est)), ko, kc)
    buf, spike = R.lipschitz_select(est, ko, kc)
    assert plan.buffered == buf and plan.interior_spike == spike


@needs_ref
@pytest.mark.parametrize("kind,n_enc,n_dec", [("encoder", 3, 0), ("decoder_only", 0, 3),
                                              ("encoder_decoder", 2, 2)])
def test_param_layout_matches_visit_params(kind, n_enc, n_dec):
    from paper_2601_09026_b200.engine import StackConfig
    cfg = StackConfig(kind=kind, d=8, heads=2, ffn=12, n_enc=n_enc, n_dec=n_dec)
    rc = R.RefStackConfig(kind=kind, d=8, heads=2, ffn=12)
    rc.n_enc, rc.n_dec = n_enc, n_dec
    st = R.RefStack(rc, 3)
    layout = L.param_layout(cfg)
    assert sum(n for *_, n in layout) == st.num_params()


def test_weight_change_rules():
    """test_lipschitz.cpp:186-255 on a d=8 encoder layout"""
    from paper_2601_09026_b200.engine import StackConfig
    cfg = StackConfig(kind="encoder", d=8, heads=2, ffn=12, n_enc=2)
    layout = L.param_layout(cfg)
    n = sum(k for *_, k in layout)
    rng = np.random.default_rng(1)
    base = rng.normal(size=n)
    for _, comp, off, k in layout:  # bias / LN-bias tensors start at zero, as at init
        if comp.endswith(".b") or comp.endswith(".bias"):
            base[off:off + k] = 0.0
    assert all(c.rel_change == 0.0 for c in L.track_weight_change(base, base, cfg))
    doubled = L.track_weight_change(2 * base, base, cfg)
    assert all(c.rel_change in (0.0, 1.0) for c in doubled)
    moved = base.copy()
    for _, comp, off, k in layout:
        if comp.endswith(".bias"):
            moved[off:off + k] = 0.25
    assert any(c.rel_change == L.kUndefinedChange for c in L.track_weight_change(moved, base, cfg))
    with pytest.raises(ContractViolation):
        L.track_weight_change(base[:-1], base, cfg)
    csv = L.weight_change_csv(doubled)
    assert csv.startswith("layer, component, rel_change\n")


# ---- the device probe --------------------------------------------------------

def _stacks():
    from paper_2601_09026_b200.engine import StackConfig
    return [
        StackConfig(kind="encoder", d=16, heads=2, ffn=32, n_enc=4),
        StackConfig(kind="decoder_only", d=16, heads=2, ffn=32, n_dec=4, buffer_open=1,
                    buffer_close=1),
        StackConfig(kind="encoder_decoder", d=16, heads=2, ffn=32, n_enc=2, n_dec=2),
        StackConfig(kind="encoder", d=64, heads=2, ffn=256, n_enc=2),
    ]


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("idx", range(4))
def test_device_probe_matches_reference(idx):
    from paper_2601_09026_b200.engine import LayerStack
    cfg = _stacks()[idx]
    st = LayerStack(cfg, seed=43)
    rc = R.RefStackConfig(kind=cfg.kind, d=cfg.d, heads=cfg.heads, ffn=cfg.ffn)
    rc.n_enc, rc.n_dec = cfg.n_enc, cfg.n_dec
    rc.buffer_open, rc.buffer_close = cfg.buffer_open, cfg.buffer_close
    ref = R.RefStack(rc, 43)
    pc = L.ProbeConfig(samples=48, delta_scale=1e-2, input_scale=1.0, seq_len=8)
    got = L.estimate_stack(st, pc, seed=47)
    assert [e.layer for e in got] == list(range(st.total_layers()))
    for e in got:
        want = R.lipschitz_estimate(ref, e.layer, pc.samples, pc.delta_scale, pc.input_scale,
                                    pc.seq_len, 47)
        # fp32 finite differences of fp32 evaluations vs the f64 reference
        assert abs(e.estimate - want) <= 2e-3 * want, (e.layer, e.estimate, want)


@pytest.mark.gpu
def test_device_probe_is_deterministic_and_layerwise():
    from paper_2601_09026_b200.engine import LayerStack
    st = LayerStack(_stacks()[0], seed=5)
    pc = L.ProbeConfig(samples=40, seq_len=4)
    a = L.estimate_stack(st, pc, seed=11)
    b = L.estimate_stack(st, pc, seed=11)
    assert [x.estimate for x in a] == [x.estimate for x in b]
    one = L.estimate_lipschitz(st, 2, pc, seed=11)
    assert one.estimate == a[2].estimate and one.layer == 2
    assert all(x.estimate > 0 for x in a)
    csv = L.lipschitz_csv(a, st)
    assert csv.startswith("layer, estimate, amplification, samples, seed\n")
    assert csv.count("\n") == st.total_layers() + 1
    rec = L.recommend_buffers(a, st, amp_threshold=2.0)
    assert rec.k_open + rec.k_close < st.total_layers()
    with pytest.raises(ValidationError):
        L.estimate_lipschitz(st, 99, pc, seed=1)
