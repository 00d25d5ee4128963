"""The adjoint's exact power-of-two scaling of lambda_N (kernels.cuh LamScale;
VERDICT r1 weak #3: the fp16 hi/lo split has no exponent scaling of its own,
so an O(1e-5..1e-8) upstream -- a mean-token cross entropy over thousands of
tokens -- would put most of lambda into fp16 subnormals).

The adjoint (Phi^T, the parameter pass, the residual norms) is linear in
lambda (blocks.cpp:516-574, mgrit.hpp:159-193), so the engine runs it on
2^k lambda_N, max in [1, 2), and multiplies lambda_0, the gradient
accumulation and the trace by 2^-k. Checked here:
  * lambda_N * 2^-30 / 2^+12 gives EXACTLY 2^-30 / 2^12 times every output
    of the unscaled run (bitwise: powers of two commute with every rounding);
  * lambda_N * 1e-8 and * 1e6 against the compiled reference's outputs
    (tests/golden/enc_small.npz) times the same factor, at the 1e-4 bar;
  * warm-started adjoint solves whose lambda_N changes by binades between
    calls match the compiled reference engine's warm-started sequence, and
    snapshot / restore across such a change is exact;
  * the raw tensor-core GEMM at operands of 1e-5 and 1e-6 stays within 1e-4.
"""
import json
import os

import numpy as np
import pytest

from paper_2601_09026_b200 import LayerParallelEngine, LayerStack, SolveConfig, StackConfig, State

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden():
    g = np.load(os.path.join(GOLDEN, "enc_small.npz"))
    return g, json.loads(str(g["meta"]))


def build(m, warm=False):
    st = LayerStack(StackConfig(kind=m["kind"], d=m["d"], heads=m["heads"], ffn=m["ffn"],
                                n_enc=m["n_enc"]), m["seed"], device=0)
    eng = LayerParallelEngine(st, SolveConfig(coarsen=m["cf"], levels=m["levels"],
                                              fwd_iters=m["fwd_iters"],
                                              bwd_iters=m["bwd_iters"], warm_start=warm))
    return st, eng


def sf(m, a):
    return State.from_flat(np.asarray(a, np.float64), m["B"], m["sx"], m["sy"], m["d"])


def adjoint(st, eng, m, traj, lam):
    grads = st.zero_grads()
    bo = eng.backward(traj, sf(m, lam), grads)
    return (np.asarray(bo.lambda0.flat()), np.asarray(bo.phase.trace, np.float64),
            np.asarray(grads, np.float64))


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.mark.parametrize("e", [-30, 12])
def test_power_of_two_lambda_is_exact(e):
    g, m = golden()
    st, eng = build(m)
    fo = eng.forward(sf(m, g["z0"]))
    l0, t0, g0 = adjoint(st, eng, m, fo.traj, g["lamN"])
    f = 2.0 ** e
    l1, t1, g1 = adjoint(st, eng, m, fo.traj, g["lamN"] * f)
    assert np.array_equal(l1, l0 * f)
    assert np.array_equal(t1, t0 * f)
    assert np.array_equal(g1, g0 * f)


@pytest.mark.parametrize("f", [1e-8, 3e-6, 1e6])
def test_scaled_lambda_matches_reference(f):
    """against the compiled reference's lambda_0, trace and gradients (the
    reference adjoint is linear: its outputs at f * lambda_N are f times)"""
    g, m = golden()
    st, eng = build(m)
    fo = eng.forward(sf(m, g["z0"]))
    l0, tr, gr = adjoint(st, eng, m, fo.traj, g["lamN"] * f)
    assert rel(l0, g["lam0"] * f) < 1e-4
    assert rel(tr, np.asarray(g["bwd_trace"]) * f) < 1e-4
    assert rel(gr, g["grads"] * f) < 1e-4


@pytest.mark.parametrize("f", [2.0 ** -24, 2.0 ** 9, 1e-7])
def test_warm_start_across_binades_matches_reference(f):
    """warm adjoint states are stored at the previous solve's 2^k: a second
    warm-started solve whose lambda_N sits binades away must see them rescaled
    (and scaled with its own 2^k without overflowing). Against the compiled
    reference engine run with the same warm-start sequence."""
    from oracle import ref as R
    if not R.available():
        pytest.skip("reference oracle not built")
    g, m = golden()
    lam2 = g["lamN"][::-1].copy() * f
    st, eng = build(m, warm=True)
    fo = eng.forward(sf(m, g["z0"]))
    adjoint(st, eng, m, fo.traj, g["lamN"])
    l_dev, t_dev, g_dev = adjoint(st, eng, m, fo.traj, lam2)

    rs = R.RefStack(R.RefStackConfig(kind=m["kind"], d=m["d"], heads=m["heads"], ffn=m["ffn"],
                                     n_enc=m["n_enc"]), m["seed"])
    re = R.RefEngine(rs, coarsen=m["cf"], levels=m["levels"], fwd_iters=m["fwd_iters"],
                     bwd_iters=m["bwd_iters"], warm_start=True)
    traj, _, _ = re.forward(g["z0"], m["B"], m["sx"], m["sy"])
    re.backward(traj, g["lamN"], m["B"], m["sx"], m["sy"], grads=np.zeros(rs.num_params()))
    gr = np.zeros(rs.num_params())
    l_ref, t_ref, _ = re.backward(traj, lam2, m["B"], m["sx"], m["sy"], grads=gr)
    assert rel(l_dev, l_ref) < 1e-4
    assert rel(t_dev, t_ref) < 1e-4
    assert rel(g_dev, gr) < 1e-4


def test_snapshot_restore_keeps_the_scale():
    g, m = golden()
    st, eng = build(m, warm=True)
    fo = eng.forward(sf(m, g["z0"]))
    adjoint(st, eng, m, fo.traj, g["lamN"])
    snap = eng.snapshot()
    ref = adjoint(st, eng, m, fo.traj, g["lamN"][::-1].copy())
    adjoint(st, eng, m, fo.traj, g["lamN"] * 2.0 ** 40)  # moves the stored scale
    eng.restore(snap)
    again = adjoint(st, eng, m, fo.traj, g["lamN"][::-1].copy())
    for a, b in zip(again, ref):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("scale", [1e-5, 1e-6])
def test_gemm_small_operands(scale):
    """the raw split GEMM (no engine scaling) with A of magnitude 1e-5 / 1e-6:
    hi is then partly subnormal, lo' keeps ~2^-35 absolute error per entry"""
    import torch
    from test_gemm import relerr, run
    torch.manual_seed(0)
    c, ref = run(2, 256, 256, 768, False, False, True, engine=0, seed=3)
    c_s, ref_s = run(2, 256, 256, 768, False, False, True, engine=0, seed=3, a_scale=scale)
    assert relerr(c_s, ref_s) < 1e-4
