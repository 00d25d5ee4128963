"""Device parity for the MGRIT hot path, through the C-ABI, against outputs of
the compiled reference (tests/golden/*.npz, made by make_golden.py) and the
float64 numpy restatement (oracle/mglp_oracle.py).

Tolerance (north star): max|device - reference| / max|reference| <= 1e-4 for
states, residual norms, lambda_0 and gradients; the device runs fp32 with
3-pass fp16-split tensor-core GEMMs (~22-bit operands, fp32 accumulation),
so observed errors are ~1e-6.
"""
import ctypes as C
import glob
import json
import os

import numpy as np
import pytest

from oracle import mglp_oracle as O
from paper_2601_09026_b200 import (LayerParallelEngine, LayerStack, SolveConfig, StackConfig,
                                   State, serial_adjoint, serial_forward)
from paper_2601_09026_b200 import _native as N

pytestmark = pytest.mark.gpu
TOL = 1e-4
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = max(float(np.abs(b).max()), 1e-300)
    return float(np.abs(a - b).max() / den)


def load(name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    return g, json.loads(str(g["meta"]))


def stack_cfg(m):
    return StackConfig(kind=m["kind"], d=m["d"], heads=m["heads"], ffn=m["ffn"], n_enc=m["n_enc"],
                       n_dec=m["n_dec"], buffer_open=m["buffer_open"],
                       buffer_close=m["buffer_close"])


def solve_cfg(m, **kw):
    c = dict(coarsen=m["cf"], levels=m["levels"], fwd_iters=m["fwd_iters"],
             bwd_iters=m["bwd_iters"], warm_start=False)
    c.update(kw)
    return SolveConfig(**c)


def build(name):
    g, m = load(name)
    st = LayerStack(stack_cfg(m), m["seed"])
    if "params" in g:
        st.set_params(g["params"])
    st_flat = lambda a: State.from_flat(a, m["B"], m["sx"], m["sy"], m["d"])  # noqa: E731
    return g, m, st, st_flat


SMALL = ["enc_small", "enc_small_3lvl", "causal_buffered", "encdec"]


@pytest.mark.parametrize("name", SMALL + ["tiny_baseline"])
def test_native_init_is_bitwise_reference_init(name):
    g, m = load(name)
    st = LayerStack(stack_cfg(m), m["seed"])
    p = np.asarray(st.params())
    assert p.size == m["n_params"]
    if "params" in g:
        assert np.array_equal(p, g["params"])
    assert float(p.sum()) == m["params_sum"]
    assert float((p * p).sum()) == m["params_sumsq"]


@pytest.mark.parametrize("name", SMALL)
def test_step_and_adjoint_step_every_layer(name):
    g, m, st, sf = build(name)
    ost = O.Stack(O.StackConfig(kind=m["kind"], d=m["d"], heads=m["heads"], ffn=m["ffn"],
                                n_enc=m["n_enc"], n_dec=m["n_dec"],
                                buffer_open=m["buffer_open"], buffer_close=m["buffer_close"]),
                  g["params"])
    z = sf(g["z0"])
    lam = sf(g["lamN"])
    oz = O.State.from_flat(g["z0"], m["B"], m["sx"], m["sy"], m["d"])
    ol = O.State.from_flat(g["lamN"], m["B"], m["sx"], m["sy"], m["d"])
    for layer in range(st.total_layers()):
        dt = 0.37
        got = st.step(layer, dt, z).flat()
        want = ost.step(layer, dt, oz).flat()
        assert rel(got, want) < 1e-5, (layer, rel(got, want))
        gr = st.zero_grads()
        got = st.adjoint_step(layer, dt, z, lam, gr, 0.5).flat()
        og = ost.zero_grads()
        want = ost.adjoint_step(layer, dt, oz, ol, og, 0.5).flat()
        assert rel(got, want) < 1e-5, (layer, rel(got, want))
        wg = O.Stack.flatten(og)
        assert rel(gr, wg) < 1e-5, (layer, rel(gr, wg))


@pytest.mark.parametrize("name", SMALL)
def test_serial_sweeps(name):
    g, m, st, sf = build(name)
    traj = serial_forward(st, sf(g["z0"]))
    T = np.stack([t.flat() for t in traj])
    assert rel(T, g["serial_traj"]) < TOL
    gr = st.zero_grads()
    lam = serial_adjoint(st, traj, sf(g["lamN"]), gr)
    L = np.stack([t.flat() for t in lam])
    assert rel(L, g["serial_lam"]) < TOL
    assert rel(gr, g["serial_grads"]) < TOL


@pytest.mark.parametrize("name", SMALL)
def test_engine_forward_backward(name):
    g, m, st, sf = build(name)
    eng = LayerParallelEngine(st, solve_cfg(m))
    fo = eng.forward(sf(g["z0"]))
    T = np.stack([t.flat() for t in fo.traj])
    assert rel(T, g["traj"]) < TOL
    assert len(fo.phase.trace) == len(g["fwd_trace"])
    assert rel(fo.phase.trace, g["fwd_trace"]) < TOL
    gr = st.zero_grads()
    bo = eng.backward(fo.traj, sf(g["lamN"]), gr)
    assert rel(bo.phase.trace, g["bwd_trace"]) < TOL
    assert rel(bo.lambda0.flat(), g["lam0"]) < TOL
    assert rel(gr, g["grads"]) < TOL


def test_engine_backward_with_host_trajectory():
    g, m, st, sf = build("enc_small")
    eng = LayerParallelEngine(st, solve_cfg(m))
    traj = [sf(t) for t in g["traj"]]  # host-provided (reference) trajectory
    gr = st.zero_grads()
    bo = eng.backward(traj, sf(g["lamN"]), gr)
    assert rel(bo.lambda0.flat(), g["lam0"]) < TOL
    assert rel(gr, g["grads"]) < TOL


def test_tiny_baseline_config():
    """BASELINE.json configs[0]: L=16, d=64, 2 heads, seq 32, batch 8, 2-level
    MGRIT c_f=4, one fwd+bwd iteration -- against the compiled reference."""
    g, m, st, sf = build("tiny_baseline")
    eng = LayerParallelEngine(st, solve_cfg(m))
    fo = eng.forward(sf(g["z0"]))
    assert rel(fo.phase.trace, g["fwd_trace"]) < TOL
    assert rel(fo.traj[-1].flat(), g["traj_last"]) < TOL
    assert rel(fo.traj[len(fo.traj) // 2].flat(), g["traj_mid"]) < TOL
    gr = st.zero_grads()
    bo = eng.backward(fo.traj, sf(g["lamN"]), gr)
    assert rel(bo.phase.trace, g["bwd_trace"]) < TOL
    assert rel(bo.lambda0.flat(), g["lam0"]) < TOL
    assert rel(gr[:4096], g["grads_head"]) < TOL
    assert abs(np.linalg.norm(gr) - g["grads_l2"][0]) / g["grads_l2"][0] < TOL
    # every one of the ~800k gradient entries: against the whole vector's max,
    # and per (layer, tensor) against that tensor's max (a tensor whose exact
    # gradient vanishes -- the attention key bias -- against its layer's)
    ref = np.asarray(g["grads"], np.float64)
    assert rel(gr, ref) < TOL
    from paper_2601_09026_b200 import lipschitz as L
    lay = L.param_layout(st.cfg)
    layer_max = {}
    for layer, comp, off, n in lay:
        layer_max[layer] = max(layer_max.get(layer, 0.0), float(np.abs(ref[off:off + n]).max()))
    for layer, comp, off, n in lay:
        r = ref[off:off + n]
        den = float(np.abs(r).max())
        den = layer_max[layer] if den < 1e-9 * layer_max[layer] else max(den, 1e-3 * layer_max[layer])
        err = float(np.abs(np.asarray(gr[off:off + n]) - r).max()) / den
        assert err < TOL, (layer, comp, err)
    traj = serial_forward(st, sf(g["z0"]))
    assert rel(traj[-1].flat(), g["serial_last"]) < TOL


def test_fixed_point_is_bitwise():
    """SURVEY 8(c) device self-test: seeded with the device's own serial
    trajectory, one V-cycle leaves every state bitwise unchanged and measures
    a residual of exactly 0 (mgrit.hpp:50-56 FAS cancellation)."""
    for name in ["enc_small", "enc_small_3lvl", "encdec"]:
        g, m, st, sf = build(name)
        eng = LayerParallelEngine(st, solve_cfg(m, cold_guess="warm", fwd_iters=1))
        eng._sync()
        z0 = sf(g["z0"])
        b, sx, sy = z0.shape
        zf = z0.flat()
        T0 = np.empty((st.total_layers() + 1, zf.size))
        N.call("mglp_serial_forward", eng.handle, b, sx, sy, N.dptr(zf), N.dptr(T0))
        N.call("mglp_engine_seed_forward_from_traj", eng.handle)
        fo = eng.forward(z0)
        assert fo.phase.trace == [0.0]
        T1 = np.stack([t.flat() for t in fo.traj])
        assert np.array_equal(T0, T1)


def test_zero_terminal_sensitivity_gives_zero_gradients():
    """test_adjoint.cpp:216-235"""
    g, m, st, sf = build("enc_small")
    eng = LayerParallelEngine(st, solve_cfg(m, fwd_iters=4, bwd_iters=2))
    fo = eng.forward(sf(g["z0"]))
    gr = st.zero_grads()
    bo = eng.backward(fo.traj, fo.traj[-1].zeros_like(), gr)
    assert np.all(gr == 0.0)
    assert np.all(bo.lambda0.flat() == 0.0)


def test_tight_solve_converges_to_serial():
    """test_adjoint.cpp:153-214 with the fp32 floor: tol 1e-6 converges and
    matches the serial sweep."""
    g, m, st, sf = build("causal_buffered")
    eng = LayerParallelEngine(st, solve_cfg(m, fwd_iters=40, bwd_iters=40, fwd_tol=1e-6,
                                            bwd_tol=1e-6))
    fo = eng.forward(sf(g["z0"]))
    assert fo.phase.converged
    T = np.stack([t.flat() for t in fo.traj])
    assert rel(T, g["serial_traj"]) < TOL
    gr = st.zero_grads()
    bo = eng.backward(fo.traj, sf(g["lamN"]), gr)
    assert bo.phase.converged
    assert rel(gr, g["serial_grads"]) < TOL
    assert rel(bo.lambda0.flat(), g["serial_lam"][0]) < TOL


def test_deterministic_and_snapshot_restore():
    g, m, st, sf = build("enc_small")
    cfg = solve_cfg(m, warm_start=True)
    a, b, c = sf(g["z0"]), sf(g["z0"] * 0.5), sf(g["z0"] * -0.3)
    probed = LayerParallelEngine(st, cfg)
    plain = LayerParallelEngine(st, solve_cfg(m, warm_start=True))
    probed.forward(a)
    probed.snapshot()
    probed.forward(b)
    probed.restore()
    got = probed.forward(c)
    plain.forward(a)
    want = plain.forward(c)
    for x, y in zip(got.traj, want.traj):
        assert np.array_equal(x.flat(), y.flat())
    # repeated identical runs are bitwise identical (no atomics, fixed orders)
    e1 = LayerParallelEngine(st, solve_cfg(m))
    e2 = LayerParallelEngine(st, solve_cfg(m))
    r1, r2 = e1.forward(a), e2.forward(a)
    g1, g2 = st.zero_grads(), st.zero_grads()
    e1.backward(r1.traj, sf(g["lamN"]), g1)
    e2.backward(r2.traj, sf(g["lamN"]), g2)
    assert np.array_equal(g1, g2)
    assert r1.phase.trace == r2.phase.trace


def test_warm_start_reuses_solution():
    """test_adjoint.cpp:311-327 (fp32: the floor is ~1e-7 relative)."""
    g, m, st, sf = build("enc_small")
    eng = LayerParallelEngine(st, solve_cfg(m, fwd_iters=6, warm_start=True))
    cold = eng.forward(sf(g["z0"]))
    warm = eng.forward(sf(g["z0"]))
    assert warm.phase.trace[0] < 1e-4 * cold.phase.trace[0]


@pytest.mark.parametrize("cfg", [(2, 1, 2, 1), (4, 2, 1, 1), (2, 3, 3, 3), (8, 2, 2, 2)])
def test_against_numpy_oracle_random_configs(cfg):
    cf, lv, fi, bi = cfg
    sc = StackConfig(kind="encoder", d=32, heads=4, ffn=64, n_enc=16)
    st = LayerStack(sc, 123)
    ost = O.Stack(O.StackConfig(kind="encoder", d=32, heads=4, ffn=64, n_enc=16),
                  np.asarray(st.params()))
    rng = np.random.default_rng(cf * 10 + lv)
    B, s = 3, 11
    z0 = rng.standard_normal(B * s * 32) * 0.5
    lam = rng.standard_normal(B * s * 32)
    eng = LayerParallelEngine(st, SolveConfig(coarsen=cf, levels=lv, fwd_iters=fi, bwd_iters=bi))
    fo = eng.forward(State.from_flat(z0, B, s, 0, 32))
    gr = st.zero_grads()
    bo = eng.backward(fo.traj, State.from_flat(lam, B, s, 0, 32), gr)
    oe = O.LayerParallelEngine(ost, O.SolveConfig(coarsen=cf, levels=lv, fwd_iters=fi,
                                                  bwd_iters=bi))
    otraj, otr, _ = oe.forward(O.State.from_flat(z0, B, s, 0, 32))
    og = ost.zero_grads()
    ol0, obtr, _ = oe.backward(otraj, O.State.from_flat(lam, B, s, 0, 32), og)
    assert rel(np.stack([t.flat() for t in fo.traj]), np.stack([t.flat() for t in otraj])) < TOL
    assert rel(fo.phase.trace, otr) < TOL
    assert rel(bo.phase.trace, obtr) < TOL
    assert rel(bo.lambda0.flat(), ol0.flat()) < TOL
    assert rel(gr, O.Stack.flatten(og)) < TOL


def test_full_width_slice_against_numpy_oracle():
    """BERT-width block (d=768, 12 heads, ffn=3072, seq 128) on a shallow
    stack: the K=768/3072 GEMMs and 128-token attention at full size."""
    sc = StackConfig(kind="encoder", d=768, heads=12, ffn=3072, n_enc=8)
    st = LayerStack(sc, 7)
    ost = O.Stack(O.StackConfig(kind="encoder", d=768, heads=12, ffn=3072, n_enc=8),
                  np.asarray(st.params()))
    rng = np.random.default_rng(3)
    B, s = 2, 128
    z0 = rng.standard_normal(B * s * 768) * 0.5
    lam = rng.standard_normal(B * s * 768)
    cfg = dict(coarsen=4, levels=2, fwd_iters=1, bwd_iters=1)
    eng = LayerParallelEngine(st, SolveConfig(**cfg))
    fo = eng.forward(State.from_flat(z0, B, s, 0, 768))
    gr = st.zero_grads()
    bo = eng.backward(fo.traj, State.from_flat(lam, B, s, 0, 768), gr)
    oe = O.LayerParallelEngine(ost, O.SolveConfig(**cfg))
    otraj, otr, _ = oe.forward(O.State.from_flat(z0, B, s, 0, 768))
    og = ost.zero_grads()
    ol0, obtr, _ = oe.backward(otraj, O.State.from_flat(lam, B, s, 0, 768), og)
    assert rel(np.stack([t.flat() for t in fo.traj]), np.stack([t.flat() for t in otraj])) < TOL
    assert rel(fo.phase.trace, otr) < TOL
    assert rel(bo.phase.trace, obtr) < TOL
    assert rel(bo.lambda0.flat(), ol0.flat()) < TOL
    assert rel(gr, O.Stack.flatten(og)) < TOL


@pytest.mark.parametrize("kind", ["encoder", "decoder_only", "encoder_decoder"])
def test_full_size_fixed_point_and_convergence(kind):
    """Size-independent properties at BASELINE sizes (d=768/512, 128-token
    sequences, batch 32): one V-cycle from the device serial trajectory is a
    bitwise fixed point; a converged MGRIT solve reproduces the serial sweep."""
    if kind == "encoder_decoder":
        sc = StackConfig(kind=kind, d=512, heads=8, ffn=2048, n_enc=8, n_dec=8)
        B, sx, sy, d = 32, 128, 128, 512
    else:
        sc = StackConfig(kind=kind, d=768, heads=12, ffn=3072, n_enc=16 if kind == "encoder" else 0,
                         n_dec=16 if kind == "decoder_only" else 0)
        B, sx, sy, d = 32, 128, 0, 768
    st = LayerStack(sc, 7)
    n = B * (sx + sy) * d
    rng = np.random.default_rng(0)
    z0 = State.from_flat(rng.standard_normal(n) * 0.5, B, sx, sy, d)
    eng = LayerParallelEngine(st, SolveConfig(coarsen=4, levels=2, fwd_iters=1, cold_guess="warm"))
    eng._sync()
    zf = z0.flat()
    T0 = np.empty((st.total_layers() + 1, zf.size))
    N.call("mglp_serial_forward", eng.handle, B, sx, sy, N.dptr(zf), N.dptr(T0))
    N.call("mglp_engine_seed_forward_from_traj", eng.handle)
    fo = eng.forward(z0)
    assert fo.phase.trace == [0.0]
    assert np.array_equal(T0, np.stack([t.flat() for t in fo.traj]))
    eng2 = LayerParallelEngine(st, SolveConfig(coarsen=4, levels=2, fwd_iters=8, warm_start=False))
    f2 = eng2.forward(z0)
    assert f2.phase.trace[-1] < 1e-5 * f2.phase.trace[0]
    assert rel(np.stack([t.flat() for t in f2.traj]), T0) < TOL
