"""Engine state contracts against the compiled reference engine
(oracle/_ref): the forward solver's warm states are independent of serial
sweeps and uploaded trajectories (adjoint.hpp:113-137 vs blocks.cpp:659-666),
parameter / mask changes invalidate the cached linearisation (the reference
recomputes everything from the current stack, adjoint.hpp:139-183),
snapshots are values (adjoint.hpp:187-206), and a captured step never
replays a stale iteration budget."""
import ctypes as C

import numpy as np
import pytest

from oracle import ref as R
from paper_2601_09026_b200 import (LayerParallelEngine, LayerStack, SolveConfig, StackConfig,
                                   State, serial_forward)
from paper_2601_09026_b200 import _native as N
from paper_2601_09026_b200.engine import ValidationError

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="reference oracle not built")]
TOL = 1e-4
D, H, F, L, B, S = 32, 2, 64, 16, 2, 9


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(float(np.abs(b).max()), 1e-300))


def pair(seed=21, **solve):
    cfg = dict(coarsen=4, levels=2, fwd_iters=1, bwd_iters=1, warm_start=True)
    cfg.update(solve)
    st = LayerStack(StackConfig(kind="encoder", d=D, heads=H, ffn=F, n_enc=L), seed)
    rs = R.RefStack(R.RefStackConfig(kind="encoder", d=D, heads=H, ffn=F, n_enc=L), seed)
    assert np.array_equal(np.asarray(st.params()), rs.get_params())
    dev = LayerParallelEngine(st, SolveConfig(**cfg))
    ref = R.RefEngine(rs, workers=2, **cfg)
    return st, rs, dev, ref


def inputs(k):
    rng = np.random.default_rng(100 + k)
    return rng.standard_normal(B * S * D) * 0.5, rng.standard_normal(B * S * D)


def sf(a):
    return State.from_flat(a, B, S, 0, D)


def test_serial_sweep_does_not_become_the_warm_start():
    st, rs, dev, ref = pair()
    za, _ = inputs(0)
    zb, _ = inputs(1)
    zc, _ = inputs(2)
    dev.forward(sf(za))
    ref.forward(za, B, S, 0)
    serial_forward(st, sf(zc))          # writes the device trajectory buffer
    rs.serial_forward(zc, B, S, 0)      # (reference: a separate vector)
    got = dev.forward(sf(zb))           # warm start from the forward solve of za
    want, wtr, _ = ref.forward(zb, B, S, 0)
    assert rel(np.stack([t.flat() for t in got.traj]), want) < TOL
    assert rel(got.phase.trace, wtr) < TOL


def test_uploaded_trajectory_does_not_become_the_warm_start():
    st, rs, dev, ref = pair()
    za, lam = inputs(0)
    zb, _ = inputs(1)
    zc, _ = inputs(2)
    dev.forward(sf(za))
    ref.forward(za, B, S, 0)
    # backward at a trajectory the caller supplies (here: the serial one of zc)
    straj = serial_forward(st, sf(zc))
    rtraj = rs.serial_forward(zc, B, S, 0)
    g = st.zero_grads()
    rg = np.zeros(rs.num_params())
    bo = dev.backward([State.from_flat(t.flat(), B, S, 0, D) for t in straj], sf(lam), g)
    rl0, rbtr, _ = ref.backward(rtraj, lam, B, S, 0, grads=rg)
    assert rel(bo.lambda0.flat(), rl0) < TOL
    assert rel(g, rg) < TOL
    got = dev.forward(sf(zb))
    want, wtr, _ = ref.forward(zb, B, S, 0)
    assert rel(np.stack([t.flat() for t in got.traj]), want) < TOL
    assert rel(got.phase.trace, wtr) < TOL


def test_set_params_between_forward_and_backward():
    """backward linearises at the given trajectory with the CURRENT parameters"""
    st, rs, dev, ref = pair(warm_start=False)
    za, lam = inputs(3)
    fo = dev.forward(sf(za))
    rtraj, _, _ = ref.forward(za, B, S, 0)
    p = np.asarray(st.params()) * 1.1
    st.set_params(p)
    rs.set_params(p)
    g = st.zero_grads()
    rg = np.zeros(rs.num_params())
    bo = dev.backward(fo.traj, sf(lam), g)   # reuses the device trajectory
    rl0, rbtr, _ = ref.backward(rtraj, lam, B, S, 0, grads=rg)
    assert rel(bo.lambda0.flat(), rl0) < TOL
    assert rel(bo.phase.trace, rbtr) < TOL
    assert rel(g, rg) < TOL


def test_snapshot_is_a_value():
    st, rs, dev, ref = pair()
    za, _ = inputs(0)
    dev.forward(sf(za))
    s1 = dev.snapshot()
    s2 = dev.snapshot()
    dev.restore(s2)
    with pytest.raises(ValidationError):
        dev.restore(s1)   # the single slot now holds s2


def test_config_change_drops_the_captured_step():
    import torch
    st, rs, dev, ref = pair(warm_start=False)
    za, lam = inputs(0)
    dev.forward(sf(za))
    h = dev.handle
    n = C.c_longlong()
    N.call("mglp_engine_set_shape", h, B, S, 0, C.byref(n))
    z = torch.zeros(n.value, device="cuda")
    z[:za.size] = torch.from_numpy(za).float()
    lm = torch.zeros_like(z)
    l0 = torch.zeros_like(z)
    N.call("mglp_engine_graph_capture", h, C.c_void_p(z.data_ptr()), C.c_void_p(lm.data_ptr()),
           C.c_void_p(l0.data_ptr()), 1)
    N.call("mglp_engine_graph_replay", h)
    d = N.SolveDesc()
    N.call("mglp_engine_get_config", h, C.byref(d))
    d.fwd_iters = 4
    N.call("mglp_engine_set_config", h, C.byref(d))
    with pytest.raises(ValidationError):
        N.call("mglp_engine_graph_replay", h)
    N.call("mglp_engine_sync", h)
