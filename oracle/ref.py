"""TEST INFRASTRUCTURE: ctypes wrapper over the compiled reference (oracle/_ref).

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
arm may import this module -- it is the checker, never the product path.

The library is the UNMODIFIED reference (/root/reference/proj/src/
{tensor,blocks,executor}.cpp) plus oracle/ref_shim.cpp, built by
oracle/Makefile. States are flat float64 arrays laid out as the reference's
State{x, y} (blocks.hpp:70-73): x [B, s_x, d] followed by y [B, s_y, d].
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libmglp_ref.so")

_dp = C.POINTER(C.c_double)
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_stack_num_params.restype = C.c_longlong
        L.ref_stack_step_size.restype = C.c_double
        L.ref_last_pair_factor.restype = C.c_double
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class RefError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


def _check(status):
    if status != 0:
        raise RefError(status, lib().ref_last_error().decode())


KIND = {"encoder": 0, "decoder_only": 1, "encoder_decoder": 2}


@dataclass
class RefStackConfig:
    kind: str = "encoder"
    d: int = 32
    heads: int = 2
    ffn: int = 64
    n_enc: int = 8
    n_dec: int = 0
    buffer_open: int = 0
    buffer_close: int = 0
    base_h: float = 1.0
    init_std: float = 0.02
    depth_scaled_init: bool = False
    dropout: float = 0.0


class RefStack:
    """The reference LayerStack (blocks.hpp:120-175)."""

    def __init__(self, cfg: RefStackConfig, seed: int):
        self.cfg = cfg
        h = C.c_void_p()
        _check(lib().ref_stack_create(
            KIND[cfg.kind], cfg.d, cfg.heads, cfg.ffn, cfg.n_enc, cfg.n_dec,
            cfg.buffer_open, cfg.buffer_close, C.c_double(cfg.base_h),
            C.c_double(cfg.init_std), int(cfg.depth_scaled_init), C.c_double(cfg.dropout),
            C.c_ulonglong(seed), C.byref(h)))
        self.h = h
        t, ib, ie, ns = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        lib().ref_stack_info(self.h, C.byref(t), C.byref(ib), C.byref(ie), C.byref(ns))
        self.total, self.ib, self.ie, self.n_split = t.value, ib.value, ie.value, ns.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_stack_destroy(self.h)
            self.h = None

    def num_params(self) -> int:
        return int(lib().ref_stack_num_params(self.h))

    def get_params(self) -> np.ndarray:
        out = np.empty(self.num_params(), np.float64)
        _check(lib().ref_stack_get_params(self.h, _ptr(out)))
        return out

    def set_params(self, flat: np.ndarray):
        flat = np.ascontiguousarray(flat, np.float64)
        assert flat.size == self.num_params()
        _check(lib().ref_stack_set_params(self.h, _ptr(flat)))

    def step_size(self, layer: int) -> float:
        return float(lib().ref_stack_step_size(self.h, layer))

    def refresh_dropout(self, seed, batch_index, b, sx, sy):
        _check(lib().ref_stack_refresh_dropout(self.h, C.c_ulonglong(seed),
                                               C.c_ulonglong(batch_index), b, sx, sy))

    def state_size(self, b, sx, sy):
        return b * (sx + sy) * self.cfg.d

    def step(self, layer, dt, z, b, sx, sy):
        z = np.ascontiguousarray(z, np.float64)
        out = np.empty_like(z)
        _check(lib().ref_stack_step(self.h, layer, C.c_double(dt), b, sx, sy, _ptr(z), _ptr(out)))
        return out

    def residual(self, layer, z, b, sx, sy):
        z = np.ascontiguousarray(z, np.float64)
        out = np.empty_like(z)
        _check(lib().ref_stack_residual(self.h, layer, b, sx, sy, _ptr(z), _ptr(out)))
        return out

    def adjoint_step(self, layer, dt, z, lam, b, sx, sy, grads=None, gscale=0.0):
        z = np.ascontiguousarray(z, np.float64)
        lam = np.ascontiguousarray(lam, np.float64)
        out = np.empty_like(z)
        _check(lib().ref_stack_adjoint_step(self.h, layer, C.c_double(dt), b, sx, sy,
                                            _ptr(z), _ptr(lam), _ptr(grads),
                                            C.c_double(gscale), _ptr(out)))
        return out

    def serial_forward(self, z0, b, sx, sy):
        z0 = np.ascontiguousarray(z0, np.float64)
        traj = np.empty((self.total + 1, z0.size), np.float64)
        _check(lib().ref_serial_forward(self.h, b, sx, sy, _ptr(z0), _ptr(traj)))
        return traj

    def serial_adjoint(self, traj, lam_n, b, sx, sy, grads=None):
        traj = np.ascontiguousarray(traj, np.float64)
        lam_n = np.ascontiguousarray(lam_n, np.float64)
        lam = np.empty_like(traj)
        _check(lib().ref_serial_adjoint(self.h, b, sx, sy, _ptr(traj), _ptr(lam_n),
                                        _ptr(lam), _ptr(grads)))
        return lam


GUESS = {"broadcast": 0, "zero": 1, "warm": 2}


class RefEngine:
    """The reference LayerParallelEngine (adjoint.hpp:99-219)."""

    def __init__(self, stack: RefStack, coarsen=2, levels=2, fwd_iters=2, bwd_iters=1,
                 fwd_tol=0.0, bwd_tol=0.0, cold_guess="broadcast", warm_start=True,
                 workers=1):
        self.stack = stack
        h = C.c_void_p()
        _check(lib().ref_engine_create(stack.h, coarsen, levels, fwd_iters, bwd_iters,
                                       C.c_double(fwd_tol), C.c_double(bwd_tol),
                                       GUESS[cold_guess], int(warm_start), workers,
                                       C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_engine_destroy(self.h)
            self.h = None

    def set_iters(self, fwd_iters, bwd_iters, fwd_tol=0.0, bwd_tol=0.0):
        lib().ref_engine_set_iters(self.h, fwd_iters, bwd_iters, C.c_double(fwd_tol),
                                   C.c_double(bwd_tol))

    def forward(self, z0, b, sx, sy, max_trace=256):
        z0 = np.ascontiguousarray(z0, np.float64)
        traj = np.empty((self.stack.total + 1, z0.size), np.float64)
        trace = np.empty(max_trace, np.float64)
        n, conv = C.c_int(), C.c_int()
        _check(lib().ref_engine_forward(self.h, b, sx, sy, _ptr(z0), _ptr(traj), _ptr(trace),
                                        max_trace, C.byref(n), C.byref(conv)))
        return traj, trace[:n.value].copy(), bool(conv.value)

    def backward(self, traj, lam_n, b, sx, sy, grads=None, max_trace=256):
        traj = np.ascontiguousarray(traj, np.float64)
        lam_n = np.ascontiguousarray(lam_n, np.float64)
        lam0 = np.empty_like(lam_n)
        trace = np.empty(max_trace, np.float64)
        n, conv = C.c_int(), C.c_int()
        _check(lib().ref_engine_backward(self.h, b, sx, sy, _ptr(traj), _ptr(lam_n),
                                         _ptr(lam0), _ptr(grads), _ptr(trace), max_trace,
                                         C.byref(n), C.byref(conv)))
        return lam0, trace[:n.value].copy(), bool(conv.value)

    def snapshot(self):
        lib().ref_engine_snapshot(self.h)

    def restore(self):
        lib().ref_engine_restore(self.h)

    def reset(self):
        lib().ref_engine_reset(self.h)


def lipschitz_estimate(stack: "RefStack", layer, samples, delta_scale, input_scale, seq_len,
                       seed) -> float:
    """estimate_lipschitz(stack, layer, cfg, seed).estimate (lipschitz.cpp:90-139)"""
    out = C.c_double()
    _check(lib().ref_lipschitz_estimate(stack.h, layer, samples, C.c_double(delta_scale),
                                        C.c_double(input_scale), seq_len, C.c_ulonglong(seed),
                                        C.byref(out)))
    return out.value


def lipschitz_select(estimates, k_open, k_close):
    """select_buffer_layers (lipschitz.cpp:151-184) -> (buffered, interior_spike)"""
    est = np.ascontiguousarray(estimates, np.float64)
    buf = (C.c_int * max(1, len(est)))()
    nb, sp = C.c_int(), C.c_int()
    _check(lib().ref_lipschitz_select(_ptr(est), len(est), k_open, k_close, buf, C.byref(nb),
                                      C.byref(sp)))
    return [buf[i] for i in range(nb.value)], bool(sp.value)


def lipschitz_recommend(amps, threshold=2.0):
    """recommend_buffers (lipschitz.cpp:219-239) -> (k_open, k_close)"""
    a = np.ascontiguousarray(amps, np.float64)
    ko, kc = C.c_int(), C.c_int()
    _check(lib().ref_lipschitz_recommend(_ptr(a), len(a), C.c_double(threshold), C.byref(ko),
                                         C.byref(kc)))
    return ko.value, kc.value


def scalar_solve(rates, h, cf, levels, z0, iters, tol=0.0, workers=1):
    rates = np.ascontiguousarray(rates, np.float64)
    n = rates.size
    states = np.empty(n + 1, np.float64)
    trace = np.empty(max(iters, 1), np.float64)
    nt, conv = C.c_int(), C.c_int()
    _check(lib().ref_scalar_solve(_ptr(rates), n, C.c_double(h), cf, levels, C.c_double(z0),
                                  iters, C.c_double(tol), workers, _ptr(states), _ptr(trace),
                                  C.byref(nt), C.byref(conv)))
    return states, trace[:nt.value].copy(), bool(conv.value)


def decide(f_fwd, f_bwd, threshold, policy, cap, fwd_iters, bwd_iters) -> int:
    d = C.c_int()
    _check(lib().ref_decide(C.c_double(f_fwd), C.c_double(f_bwd), C.c_double(threshold),
                            policy, cap, fwd_iters, bwd_iters, C.byref(d)))
    return d.value


def last_pair_factor(trace) -> float:
    t = np.ascontiguousarray(trace, np.float64)
    return float(lib().ref_last_pair_factor(_ptr(t), t.size))


def gaussian_fill(seed, a, b, n, scale=1.0):
    """scale * rng::gaussian(seed, a, b, i) for i < n (the bench z0 draw, main.cpp:121-128)."""
    out = np.empty(n, np.float64)
    lib().ref_gaussian_fill(C.c_ulonglong(seed), C.c_ulonglong(a), C.c_ulonglong(b),
                            C.c_double(scale), _ptr(out), C.c_longlong(n))
    return out


def gaussian_fill_flat(seed, a, n, scale=1.0):
    """scale * rng::gaussian(seed, a, i) (testutil::random_tensor, test_util.hpp:89-95)."""
    out = np.empty(n, np.float64)
    lib().ref_gaussian_fill_flat(C.c_ulonglong(seed), C.c_ulonglong(a), C.c_double(scale),
                                 _ptr(out), C.c_longlong(n))
    return out


# ---- training edge: make_batch, Model init, run_training -----------
TASK_KIND = {"copy_sequence": 0, "token_classification": 1, "tiny_translation": 2}
OPT_KIND = {"sgd": 0, "adam": 1, "adamw": 2}
MODE = {"serial": 0, "layer_parallel": 1, "switching": 2}
GUESS = {"broadcast": 0, "zero": 1, "warm": 2}


def _task_arr(task):
    return np.array([TASK_KIND[task.kind], task.vocab, task.seq_len, task.train_size,
                     task.val_size, task.seed], dtype=np.float64)


def _model_arr(m):
    s = m.stack
    return np.array([KIND[s.kind], s.d, s.heads, s.ffn, s.n_enc, s.n_dec, s.buffer_open,
                     s.buffer_close, s.base_h, s.init_std, float(s.depth_scaled_init), s.dropout,
                     m.vocab, m.max_seq], dtype=np.float64)


def _train_arr(t):
    so, ind, o = t.solve, t.indicator, t.opt
    return np.array([MODE[t.mode], OPT_KIND[o.kind], o.lr, o.beta1, o.beta2, o.eps,
                     o.weight_decay, o.momentum, so.coarsen, so.levels, so.fwd_iters,
                     so.bwd_iters, so.fwd_tol, so.bwd_tol, GUESS[so.cold_guess],
                     float(so.warm_start), ind.probe_period, ind.threshold, ind.policy,
                     ind.max_iter_cap, float(ind.use_probe_gradient), t.batch_size, t.epochs,
                     t.seed, t.manual_switch_batch, t.val_every], dtype=np.float64)


def make_batch(task, split, start, batch):
    """tasks.cpp:45-89 -> (src, tgt_in or None, tgt_out) int32 [batch*seq]"""
    n = batch * task.seq_len
    src, tin, tout = (np.zeros(n, dtype=np.int32) for _ in range(3))
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
    _check(lib().ref_make_batch(TASK_KIND[task.kind], task.vocab, task.seq_len, task.train_size,
                                task.val_size, C.c_ulonglong(task.seed), split,
                                C.c_longlong(start), batch, ip(src), ip(tin), ip(tout)))
    return src, (tin if task.kind == "tiny_translation" else None), tout


def model_params(mcfg, seed):
    """Model(mcfg, seed).param_tensors() (model.cpp:50-92) -> (flat, shapes)"""
    m = _model_arr(mcfg)
    n, k = C.c_longlong(), C.c_longlong()
    _check(lib().ref_model_params(_ptr(m), C.c_ulonglong(seed), None, C.byref(n), None,
                                  C.byref(k)))
    flat = np.zeros(n.value)
    sh = np.zeros(k.value, dtype=np.int64)
    _check(lib().ref_model_params(_ptr(m), C.c_ulonglong(seed), _ptr(flat), C.byref(n),
                                  sh.ctypes.data_as(C.POINTER(C.c_longlong)), C.byref(k)))
    shapes, i = [], 0
    while i < len(sh):
        r = int(sh[i])
        shapes.append(tuple(int(x) for x in sh[i + 1:i + 1 + r]))
        i += 1 + r
    return flat, shapes


def config_echo(task, mcfg, tcfg) -> str:
    t, m, r = _task_arr(task), _model_arr(mcfg), _train_arr(tcfg)
    n = C.c_longlong()
    buf = C.create_string_buffer(4096)
    _check(lib().ref_config_echo(_ptr(t), _ptr(m), _ptr(r), buf, 4096, C.byref(n)))
    return buf.raw[: n.value].decode()


def run_training(task, mcfg, tcfg, start_state: bytes = b""):
    """run_training (training.cpp:348-360) -> dict(csv, final_state,
    switch_state, switch_batch)"""
    t, m, r = _task_arr(task), _model_arr(mcfg), _train_arr(tcfg)
    L = lib()
    csv_len, st_len, sw_len, sw_b = (C.c_longlong() for _ in range(4))
    args = (_ptr(t), _ptr(m), _ptr(r), start_state or None, C.c_longlong(len(start_state or b"")))
    _check(L.ref_run_training(*args, None, 0, C.byref(csv_len), None, 0, C.byref(st_len), None,
                              C.byref(sw_len), C.byref(sw_b)))
    # the run is deterministic: re-run with buffers sized from the first call
    cap = max(st_len.value, sw_len.value)
    csv = C.create_string_buffer(csv_len.value + 1)
    st = C.create_string_buffer(cap + 1)
    sw = C.create_string_buffer(cap + 1)
    _check(L.ref_run_training(*args, csv, csv_len.value + 1, C.byref(csv_len), st, cap + 1,
                              C.byref(st_len), sw, C.byref(sw_len), C.byref(sw_b)))
    return {"csv": csv.raw[: csv_len.value].decode(), "final_state": st.raw[: st_len.value],
            "switch_state": sw.raw[: sw_len.value], "switch_batch": sw_b.value}
