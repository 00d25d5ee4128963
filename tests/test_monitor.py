"""Gradient-bias monitor on the device (controller.hpp:32-166; VERDICT r1
missing #3 / weak #4): budgets, decisions, switch flag and the report log in
device memory, record() as one kernel on the device-resident traces.

  * factors / decisions / budget updates of the device record() against the
    compiled reference's last_pair_factor and decide (oracle/_ref);
  * a CUDA graph captured with gated cycles follows device budget changes
    without recapture (bitwise equal to eager solves at that budget), and a
    budget above the captured cycles fails loudly;
  * the switching trainer against the reference's run_training for
    test_training.cpp:151-204: threshold 1e-12 trips kSwitchSerial at the
    first probe and the tail replays bitwise; measurement-only probes leave
    the update stream untouched; probe-gradient rows run the doubled budget.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle import ref as R
from paper_2601_09026_b200 import _native as N
from paper_2601_09026_b200 import training as T
from paper_2601_09026_b200.controller import (POLICY_INCREASE, POLICY_SWITCH, DeviceMonitor,
                                              IndicatorConfig)
from paper_2601_09026_b200.engine import (LayerParallelEngine, LayerStack, SolveConfig,
                                          StackConfig, State)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="reference oracle not built")]
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_engine(fwd_iters=2, bwd_iters=2, warm=False):
    g = np.load(os.path.join(GOLDEN, "enc_small.npz"))
    m = json.loads(str(g["meta"]))
    st = LayerStack(StackConfig(kind=m["kind"], d=m["d"], heads=m["heads"], ffn=m["ffn"],
                                n_enc=m["n_enc"]), m["seed"], device=0)
    eng = LayerParallelEngine(st, SolveConfig(coarsen=m["cf"], levels=m["levels"],
                                              fwd_iters=fwd_iters, bwd_iters=bwd_iters,
                                              warm_start=warm))
    sf = lambda a: State.from_flat(a, m["B"], m["sx"], m["sy"], m["d"])  # noqa: E731
    return g, m, st, eng, sf


def read(h):
    sw, dec, fi, bi, uf, ub = (C.c_int() for _ in range(6))
    ff, bf = C.c_double(), C.c_double()
    N.call("mglp_engine_monitor_read", h, C.byref(sw), C.byref(dec), C.byref(ff), C.byref(bf),
           C.byref(fi), C.byref(bi), C.byref(uf), C.byref(ub))
    return dict(switched=sw.value, decision=dec.value, ff=ff.value, bf=bf.value,
                budget=(fi.value, bi.value), used=(uf.value, ub.value))


@pytest.mark.parametrize("thr,policy,cap", [(1e-12, POLICY_INCREASE, 16),
                                            (1e-12, POLICY_SWITCH, 16),
                                            (1e-12, POLICY_INCREASE, 2),
                                            (1e9, POLICY_INCREASE, 16)])
def test_record_matches_reference_decide(thr, policy, cap):
    g, m, st, eng, sf = golden_engine()
    mon = DeviceMonitor(IndicatorConfig(threshold=thr, policy=policy, max_iter_cap=cap),
                        eng.handle, trainer=False)
    fo = eng.forward(sf(g["z0"]))
    bo = eng.backward(fo.traj, sf(g["lamN"]), st.zero_grads())
    rep = mon.record_engine(7)
    f_ref = R.last_pair_factor(fo.phase.trace)
    b_ref = R.last_pair_factor(bo.phase.trace)
    assert rep.fwd_factor == f_ref and rep.bwd_factor == b_ref  # same f64 division
    dec = R.decide(f_ref, b_ref, thr, policy, cap, 2, 2)
    assert rep.decision == dec
    s = read(eng.handle)
    assert s["used"] == (2, 2)
    if dec == 1:
        assert s["budget"] == (min(4, cap), min(4, cap))
    else:
        assert s["budget"] == (2, 2)
    assert s["switched"] == int(dec == 2) == int(mon.switched())
    r = mon.reports
    assert len(r) == 1 and r[0].batch == 7 and r[0].decision == dec


def test_device_budget_drives_the_solves():
    """after an increase decision the next solves run the doubled budget
    (their traces grow) without any host-side config change"""
    g, m, st, eng, sf = golden_engine(1, 1)
    DeviceMonitor(IndicatorConfig(threshold=1e-12, policy=POLICY_INCREASE, max_iter_cap=8),
                  eng.handle, trainer=False)
    fo = eng.forward(sf(g["z0"]))
    eng.backward(fo.traj, sf(g["lamN"]), st.zero_grads())
    # one-cycle traces: factor 0 -> keep
    N.call("mglp_monitor_record", eng.handle, 0, None)
    assert read(eng.handle)["decision"] == 0
    N.call("mglp_engine_monitor_probe", eng.handle, 1)  # ProbeScope: 2 + 2
    fo = eng.forward(sf(g["z0"]), want_traj=True)
    # eng.forward re-syncs the Python config (1, 1); the device budget wins
    assert len(fo.phase.trace) == 2
    eng.backward(fo.traj, sf(g["lamN"]), st.zero_grads())
    N.call("mglp_engine_monitor_probe", eng.handle, 0)
    N.call("mglp_monitor_record", eng.handle, 1, None)
    s = read(eng.handle)
    assert s["used"] == (2, 2) and s["decision"] == 1 and s["budget"] == (2, 2)


def test_gated_graph_follows_device_budget():
    import torch
    g, m, st, eng, sf = golden_engine(1, 1)
    h = eng.handle
    DeviceMonitor(IndicatorConfig(threshold=1e9, max_iter_cap=16), h, trainer=False)
    ns = C.c_longlong()
    N.call("mglp_engine_set_shape", h, m["B"], m["sx"], m["sy"], C.byref(ns))
    n = m["B"] * (m["sx"] + m["sy"]) * m["d"]
    z0 = torch.zeros(ns.value, device="cuda")
    lam = torch.zeros_like(z0)
    lam0 = torch.zeros_like(z0)
    z0[:n] = torch.from_numpy(g["z0"]).float()
    lam[:n] = torch.from_numpy(g["lamN"]).float()
    p = np.ascontiguousarray(st.params())
    N.call("mglp_engine_set_params", h, N.dptr(p), p.size)
    N.call("mglp_engine_capture_cycles", h, 4)
    N.call("mglp_engine_graph_capture", h, C.c_void_p(z0.data_ptr()), C.c_void_p(lam.data_ptr()),
           C.c_void_p(lam0.data_ptr()), 1)

    def traces():
        tr = np.empty(64)
        nt, cv = C.c_int(), C.c_int()
        N.call("mglp_engine_trace", h, 0, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
        f = tr[:nt.value].copy()
        N.call("mglp_engine_trace", h, 1, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
        return f, tr[:nt.value].copy()

    def set_budget(f, b):
        sd = N.SolveDesc()
        N.call("mglp_engine_get_config", h, C.byref(sd))
        sd.fwd_iters, sd.bwd_iters = f, b
        N.call("mglp_engine_set_config", h, C.byref(sd))

    out = {}
    for f, b in [(1, 1), (3, 2), (4, 4)]:
        set_budget(f, b)
        N.call("mglp_engine_graph_replay", h)  # same graph, no recapture
        N.call("mglp_engine_sync", h)
        ft, bt = traces()
        # the budget, or fewer cycles when a solve converges exactly (tol 0:
        # this small stack's exactness front reaches the end after 3 cycles)
        assert 1 <= len(ft) <= f and 1 <= len(bt) <= b
        assert len(ft) == f or ft[-1] == 0.0
        out[(f, b)] = (ft, bt, lam0.clone())
    # eager solves at the same budgets: bitwise the gated replays
    N.call("mglp_engine_capture_cycles", h, 0)
    for (f, b), (ft, bt, l0) in out.items():
        set_budget(f, b)
        N.call("mglp_engine_forward_device", h, C.c_void_p(z0.data_ptr()))
        N.call("mglp_engine_backward_device", h, C.c_void_p(lam.data_ptr()),
               C.c_void_p(lam0.data_ptr()), 1)
        N.call("mglp_engine_sync", h)
        e_ft, e_bt = traces()
        assert np.array_equal(e_ft, ft) and np.array_equal(e_bt, bt)
        assert torch.equal(lam0, l0)
    # a budget beyond the captured cycles is refused, not truncated
    N.call("mglp_engine_capture_cycles", h, 4)
    N.call("mglp_engine_graph_capture", h, C.c_void_p(z0.data_ptr()), C.c_void_p(lam.data_ptr()),
           C.c_void_p(lam0.data_ptr()), 1)
    set_budget(8, 1)
    N.call("mglp_engine_graph_replay", h)
    with pytest.raises(N.ContractViolation):
        traces()


# ---- the switching trainer against the reference's run_training ----------------------
def classification(mode="switching", **ind):
    stack = StackConfig(kind="encoder", d=32, heads=2, ffn=64, n_enc=8)
    tk = T.TaskSpec(kind="token_classification", vocab=16, seq_len=8, train_size=16,
                    val_size=8, seed=1)
    mc = T.ModelConfig(stack=stack, vocab=16, max_seq=8)
    tc = T.TrainConfig(mode=mode, solve=SolveConfig(coarsen=2, levels=2, fwd_iters=2,
                                                    bwd_iters=1),
                       batch_size=4, epochs=2, seed=7, val_every=2,
                       indicator=IndicatorConfig(**ind))
    return tk, mc, tc


def rows(csv):
    out = []
    for line in csv.strip().splitlines()[1:]:
        f = [x.strip() for x in line.split(",")]
        out.append(dict(batch=int(f[0]), loss=float(f[1]), val=float(f[2]), mode=f[3],
                        fi=int(f[4]), bi=int(f[5]), ff=float(f[6]), bf=float(f[7])))
    return out


def compare(res, ref):
    rr = rows(ref["csv"])
    dr = rows(res.csv)
    assert [r["mode"] for r in dr] == [r["mode"] for r in rr]
    assert [(r["fi"], r["bi"]) for r in dr] == [(r["fi"], r["bi"]) for r in rr]
    for d, r in zip(dr, rr):
        assert abs(d["loss"] - r["loss"]) <= 1e-4 * abs(r["loss"]), (d, r)
        for k in ("ff", "bf"):
            assert abs(d[k] - r[k]) <= 1e-4 * max(abs(r[k]), 1e-12), (k, d, r)
    return dr, rr


def test_indicator_handover_matches_reference():
    """test_training.cpp:151-174 on the device monitor"""
    tk, mc, tc = classification(probe_period=2, threshold=1e-12, policy=POLICY_SWITCH)
    ref = R.run_training(tk, mc, tc)
    tr = T.Trainer(tk, mc, tc)
    res = tr.run()
    assert res.switched and res.switch_batch >= 1
    assert res.switch_batch == ref["switch_batch"]
    reps = res.reports
    assert reps and reps[-1].decision == 2
    assert all(r.decision != 2 for r in reps[:-1])
    for r in res.rows:
        if r.batch >= res.switch_batch:
            assert r.mode == "serial"
    compare(res, ref)
    out = T.switching_replay(tk, mc, tc)
    assert out.switched and out.losses_match and out.state_matches


def test_measurement_only_probes_leave_updates_untouched():
    """test_training.cpp:176-192: threshold 1e9, use_probe_gradient = false --
    bitwise the same losses and final state as the unmonitored run"""
    tk, mc, tc = classification(mode="layer_parallel")
    plain = T.run_training(tk, mc, tc)
    tk, mc, tc = classification(probe_period=2, threshold=1e9, use_probe_gradient=False)
    probed = T.run_training(tk, mc, tc)
    assert not probed.switched
    assert [r.batch for r in probed.reports] == [0, 2, 4, 6]
    assert [np.float64(r.loss).tobytes() for r in plain.rows] == \
        [np.float64(r.loss).tobytes() for r in probed.rows]
    assert plain.final_state == probed.final_state
    compare(probed, R.run_training(tk, mc, tc))


def test_probe_gradient_rows_run_the_doubled_budget():
    """test_training.cpp:194-204"""
    tk, mc, tc = classification(probe_period=4, threshold=1e9, use_probe_gradient=True)
    res = T.run_training(tk, mc, tc)
    assert (res.rows[0].fwd_iters, res.rows[0].bwd_iters) == (4, 2)
    assert (res.rows[1].fwd_iters, res.rows[1].bwd_iters) == (2, 1)
    compare(res, R.run_training(tk, mc, tc))


def test_increase_policy_budget_growth_matches_reference():
    """kIncreaseIterations: the device doubles the budgets (capped at 4) at
    every probe until the cap, then switches -- rows, budgets, factors and
    losses against the reference"""
    tk, mc, tc = classification(probe_period=2, threshold=1e-12, policy=POLICY_INCREASE,
                                max_iter_cap=4)
    ref = R.run_training(tk, mc, tc)
    res = T.run_training(tk, mc, tc)
    compare(res, ref)
    assert res.switched == (ref["switch_batch"] >= 0)
