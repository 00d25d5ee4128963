"""No silent fp16 overflow on the split tensor-core path (gemm_tc.cu header):
a finite operand value with |x| >= 65520 raises ContractViolation from the
engine -- now that the forward and dgrad GEMM operands are produced
pre-split, the check sits in their producers (LayerNorm, attention and GELU
epilogues, the upstream pack, the weight pack) instead of the GEMM
converters. d = 64, dh = 32, ffn = 128: every pre-split path is active."""
import numpy as np
import pytest

from paper_2601_09026_b200 import LayerParallelEngine, LayerStack, SolveConfig, StackConfig, State
from paper_2601_09026_b200 import lipschitz as L
from paper_2601_09026_b200._native import ContractViolation

pytestmark = pytest.mark.gpu

B, S, D = 2, 16, 64


def make(scale_comp=None, value=None):
    cfg = StackConfig(kind="encoder", d=D, heads=2, ffn=128, n_enc=4)
    st = LayerStack(cfg, 3, device=0)
    if scale_comp is not None:
        p = np.asarray(st.params()).copy()
        for layer, comp, off, n in L.param_layout(cfg):
            if layer == 1 and comp == scale_comp:
                p[off:off + n] = value
        st.set_params(p)
    eng = LayerParallelEngine(st, SolveConfig(coarsen=2, levels=2, fwd_iters=1, bwd_iters=1,
                                              warm_start=False))
    return st, eng


def state(seed, scale):
    rng = np.random.default_rng(seed)
    return State.from_flat((rng.standard_normal(B * S * D) * scale).astype(np.float32), B, S, 0, D)


def test_clean_run_passes():
    st, eng = make()
    fo = eng.forward(state(0, 0.5))
    eng.backward(fo.traj, state(1, 1.0), st.zero_grads())


def test_layernorm_output_beyond_fp16_raises():
    # LN2 gain 1e6: the MLP-in operand (LayerNorm output, written pre-split)
    st, eng = make("ln2.gain", 1e6)
    with pytest.raises(ContractViolation):
        eng.forward(state(0, 0.5))


def test_weight_beyond_fp16_raises():
    st, eng = make("mlp.in.w", 1e5)  # the pre-split weight pack
    with pytest.raises(ContractViolation):
        eng.forward(state(0, 0.5))


def test_large_upstream_is_rescaled_not_overflowed():
    """lambda_N of 1e6 used to overflow the upstream pack; the adjoint now runs
    on 2^k lambda_N (LamScale) and returns the exact linear multiple"""
    st, eng = make()
    fo = eng.forward(state(0, 0.5))
    g1, g2 = st.zero_grads(), st.zero_grads()
    b1 = eng.backward(fo.traj, state(1, 1.0), g1)
    b2 = eng.backward(fo.traj, state(1, 2.0 ** 20), g2)
    assert np.array_equal(np.asarray(b2.lambda0.flat()), np.asarray(b1.lambda0.flat()) * 2.0 ** 20)
    assert np.array_equal(np.asarray(g2), np.asarray(g1) * 2.0 ** 20)


def test_upstream_growth_beyond_fp16_raises():
    """the scaling normalises lambda_N only: an adjoint that itself grows past
    the fp16 range inside the stack still raises (MLP-out weight 5e4: the
    dgrad of the MLP branch multiplies the upstream by ~|W| * sqrt(d))"""
    st, eng = make("mlp.out.w", 5e4)
    with pytest.raises(ContractViolation):
        fo = eng.forward(state(0, 0.5))
        eng.backward(fo.traj, state(1, 1.0), st.zero_grads())
