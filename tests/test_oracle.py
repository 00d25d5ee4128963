"""Pins the float64 numpy oracle (oracle/mglp_oracle.py) against the compiled
reference (oracle/_ref) and the committed golden fixtures, and re-checks the
reference's own known answers for the solver (test_mgrit.cpp)."""
import glob
import json
import os

import numpy as np
import pytest

from oracle import mglp_oracle as O
from oracle import ref as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = max(np.abs(b).max(), 1e-300)
    return float(np.abs(a - b).max() / den)


CASES = [
    ("encoder", 8, 0, 0, 0, 0, 2, 2, 2, 1),
    ("encoder", 8, 0, 0, 0, 0, 2, 3, 3, 2),
    ("decoder_only", 0, 10, 1, 1, 0, 2, 2, 2, 1),
    ("encoder_decoder", 4, 4, 0, 0, 4, 2, 2, 2, 1),
    ("encoder", 16, 0, 0, 0, 0, 4, 2, 1, 1),
    ("decoder_only", 0, 16, 0, 0, 0, 4, 2, 2, 2),
]


@needs_ref
@pytest.mark.parametrize("case", CASES)
def test_numpy_oracle_matches_reference(case):
    kind, ne, nd, bo, bc, sy, cf, lv, fi, bi = case
    rc = R.RefStackConfig(kind=kind, d=8, heads=2, ffn=12, n_enc=ne, n_dec=nd, buffer_open=bo,
                          buffer_close=bc)
    rs = R.RefStack(rc, 9)
    st = O.Stack(O.StackConfig(kind=kind, d=8, heads=2, ffn=12, n_enc=ne, n_dec=nd,
                               buffer_open=bo, buffer_close=bc), rs.get_params())
    B, sx = 2, 5
    n = B * (sx + sy) * 8
    z0 = R.gaussian_fill_flat(930, 6, n, 0.5)
    lam = R.gaussian_fill_flat(931, 6, n, 1.0)
    e = R.RefEngine(rs, coarsen=cf, levels=lv, fwd_iters=fi, bwd_iters=bi, workers=2)
    traj, tr, _ = e.forward(z0, B, sx, sy)
    g = np.zeros(rs.num_params())
    l0, btr, _ = e.backward(traj, lam, B, sx, sy, grads=g)
    oe = O.LayerParallelEngine(st, O.SolveConfig(coarsen=cf, levels=lv, fwd_iters=fi,
                                                 bwd_iters=bi))
    otraj, otr, _ = oe.forward(O.State.from_flat(z0, B, sx, sy, 8))
    og = st.zero_grads()
    ol0, obtr, _ = oe.backward(otraj, O.State.from_flat(lam, B, sx, sy, 8), og)
    assert rel(np.stack([s.flat() for s in otraj]), traj) < 1e-12
    assert rel(otr, tr) < 1e-12
    assert rel(obtr, btr) < 1e-12
    assert rel(ol0.flat(), l0) < 1e-12
    assert rel(O.Stack.flatten(og), g) < 1e-12


@needs_ref
def test_phi_count_per_cycle():
    """a 2-level cycle costs 4N evaluations, 3-level 4N + 3N/c_f."""
    for n, cf, lv, want in [(64, 4, 2, 256), (128, 4, 3, 608), (64, 8, 2, 256), (16, 4, 2, 64)]:
        s = O.MgritSolver(O.ScalarLinearSystem([-0.5] * n, 1.0, cf), n, cf, lv)
        s.set_initial_condition(1.0)
        s.apply_initial_guess("broadcast")
        s.v_cycle()
        assert s.phi_calls == want


def scalar(cf, n, rate=-0.5, levels=2):
    s = O.MgritSolver(O.ScalarLinearSystem([rate] * n, 1.0, cf), n, cf, levels)
    s.set_initial_condition(1.0)
    s.apply_initial_guess("broadcast")
    return s


def test_known_answer_finite_termination():
    """test_mgrit.cpp:288-315: broadcast start reaches the serial solution
    bitwise after exactly 16 (c_f=2) / 8 (c_f=4) cycles."""
    for cf, want in [(2, 16), (4, 8)]:
        sys_ = O.ScalarLinearSystem([-0.5] * 64, 1.0, cf)
        serial = [1.0]
        for j in range(64):
            serial.append(sys_.phi(0, j, serial[-1]))
        s = scalar(cf, 64)
        reached = None
        for c in range(1, 40):
            s.v_cycle()
            if s.states(0) == serial:
                reached = c
                break
        assert reached == want


def test_known_answer_fixed_point_and_front():
    """test_mgrit.cpp:243-254 and 270-286."""
    sys_ = O.ScalarLinearSystem([-0.5] * 64, 1.0, 2)
    serial = [1.0]
    for j in range(64):
        serial.append(sys_.phi(0, j, serial[-1]))
    for levels in (2, 3):
        s = O.MgritSolver(sys_, 64, 2, levels)
        s.lv[0].v = list(serial)
        assert s.v_cycle() == 0.0
        assert s.states(0) == serial
    for cf in (2, 4):
        sys_ = O.ScalarLinearSystem([-0.5] * 64, 1.0, cf)
        serial = [1.0]
        for j in range(64):
            serial.append(sys_.phi(0, j, serial[-1]))
        s = scalar(cf, 64)
        for sweep in range(1, 6):
            s.fcf_relax(0)
            j = -1
            while j + 1 < 65 and s.states(0)[j + 1] == serial[j + 1]:
                j += 1
            assert j == min((sweep + 1) * cf - 1, 64)


@needs_ref
def test_scalar_solver_bitwise_vs_reference():
    rates = [-0.75 + 0.015 * i for i in range(32)]
    for cf, lv, it in [(2, 2, 5), (2, 3, 4), (4, 2, 3)]:
        st, tr, conv = R.scalar_solve(rates, 1.0, cf, lv, 1.0, it)
        s = O.MgritSolver(O.ScalarLinearSystem(rates, 1.0, cf), 32, cf, lv)
        s.set_initial_condition(1.0)
        s.apply_initial_guess("broadcast")
        otr, _ = s.solve_forward(it, 0.0)
        assert s.states(0) == list(st)
        assert otr == list(tr)


@needs_ref
def test_controller_matches_reference():
    for ff, bf in [(0.5, 0.2), (1.5, 0.1), (0.1, 2.0), (1.0, 1.0)]:
        for policy in (0, 1):
            for fi, bi in [(2, 1), (16, 16), (16, 4)]:
                want = R.decide(ff, bf, 1.0, policy, 16, fi, bi)
                assert O.decide(ff, bf, 1.0, policy == 1, 16, fi, bi) == want
    for t in ([], [1.0], [4.0, 2.0], [5.0, 1.0, 0.0], [3.0, 0.0, 0.0], [1.0, 3.0]):
        assert O.last_pair_factor(t) == R.last_pair_factor(t)


def _golden_files():
    # deep_*.npz / bench_*.npz are outputs OF the numpy oracle (make_deep.py);
    # the oracle is pinned at their layer shapes by test_oracle_full_width_layers
    return sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith(("deep_", "bench_")))


@pytest.mark.parametrize("path", _golden_files())
def test_oracle_reproduces_golden(path):
    """The committed fixtures (made by tests/golden/make_golden.py from the
    compiled reference) are reproduced by the numpy restatement."""
    g = np.load(path)
    meta = json.loads(str(g["meta"]))
    if meta.get("big"):
        pytest.skip("large fixture: checked against the device only")
    sc = O.StackConfig(kind=meta["kind"], d=meta["d"], heads=meta["heads"], ffn=meta["ffn"],
                       n_enc=meta["n_enc"], n_dec=meta["n_dec"],
                       buffer_open=meta["buffer_open"], buffer_close=meta["buffer_close"])
    st = O.Stack(sc, g["params"])
    B, sx, sy, d = meta["B"], meta["sx"], meta["sy"], meta["d"]
    oe = O.LayerParallelEngine(st, O.SolveConfig(coarsen=meta["cf"], levels=meta["levels"],
                                                 fwd_iters=meta["fwd_iters"],
                                                 bwd_iters=meta["bwd_iters"],
                                                 warm_start=False))
    traj, tr, _ = oe.forward(O.State.from_flat(g["z0"], B, sx, sy, d))
    gr = st.zero_grads()
    l0, btr, _ = oe.backward(traj, O.State.from_flat(g["lamN"], B, sx, sy, d), gr)
    assert rel(np.stack([s.flat() for s in traj]), g["traj"]) < 1e-12
    assert rel(tr, g["fwd_trace"]) < 1e-12
    assert rel(btr, g["bwd_trace"]) < 1e-12
    assert rel(l0.flat(), g["lam0"]) < 1e-12
    assert rel(O.Stack.flatten(gr), g["grads"]) < 1e-12


@pytest.mark.skipif(not R.available(), reason="reference oracle not built")
@pytest.mark.parametrize("shape", [("encoder", 768, 12, 3072, 20, 0),
                                   ("decoder_only", 768, 12, 3072, 24, 0),
                                   ("encoder_decoder", 512, 8, 2048, 12, 10)])
def test_oracle_full_width_layers(shape):
    """Pins the numpy restatement at the deep fixtures' layer widths (d=768 /
    512, 12 / 8 heads, ffn=4d; encoder, causal, cross-attention) against the
    compiled reference: LayerStack::step and ::adjoint_step with gradients
    (blocks.cpp:509-574) on a short sequence (the scalar reference costs
    ~1 s per full-length layer)."""
    kind, d, H, ffn, sx, sy = shape
    n_enc, n_dec = {"encoder": (2, 0), "decoder_only": (0, 2), "encoder_decoder": (1, 1)}[kind]
    rs = R.RefStack(R.RefStackConfig(kind=kind, d=d, heads=H, ffn=ffn, n_enc=n_enc,
                                     n_dec=n_dec), 7)
    st = O.Stack(O.StackConfig(kind=kind, d=d, heads=H, ffn=ffn, n_enc=n_enc, n_dec=n_dec),
                 rs.get_params())
    n = sx * d + sy * d
    z = R.gaussian_fill(7, 6, 7, n, 0.5)
    lam = R.gaussian_fill(8, 6, 8, n, 1.0)
    for layer in range(st.total):
        want = rs.step(layer, 0.5, z, 1, sx, sy)
        got = st.step(layer, 0.5, O.State.from_flat(z, 1, sx, sy, d)).flat()
        assert rel(got, want) < 1e-12
        rg = np.zeros(rs.num_params())
        want = rs.adjoint_step(layer, 0.5, z, lam, 1, sx, sy, grads=rg, gscale=0.25)
        og = st.zero_grads()
        got = st.adjoint_step(layer, 0.5, O.State.from_flat(z, 1, sx, sy, d),
                              O.State.from_flat(lam, 1, sx, sy, d), og, 0.25).flat()
        assert rel(got, want) < 1e-12
        assert rel(O.Stack.flatten(og), rg) < 1e-12
