"""Host-side mirror of the reference's solver / layer / engine API over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj:
  StackConfig, LayerStack        include/mglp/blocks.hpp:100-175
  State                          blocks.hpp:70-73 (x [B,s_x,d], y [B,s_y,d] or None)
  serial_forward/serial_adjoint  blocks.hpp:190-199
  SolveConfig, PhaseTrace,
  ForwardOutcome, BackwardOutcome,
  LayerParallelEngine            include/mglp/adjoint.hpp:70-219
Everything numeric runs in libmglp_cuda.so on the GPU; this module only
marshals float64 host arrays across the boundary.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N
from ._native import ContractViolation, ValidationError  # noqa: F401

KINDS = {"encoder": 0, "decoder_only": 1, "encoder_decoder": 2}
GUESSES = {"broadcast": 0, "zero": 1, "warm": 2}


@dataclass
class StackConfig:
    """blocks.hpp:100-114."""
    kind: str = "encoder"
    d: int = 32
    heads: int = 2
    ffn: int = 64
    n_enc: int = 8
    n_dec: int = 0
    buffer_open: int = 0
    buffer_close: int = 0
    ln_eps: float = 1e-5
    base_h: float = 1.0
    dropout: float = 0.0
    init_std: float = 0.02
    depth_scaled_init: bool = False

    def desc(self) -> N.StackDesc:
        if self.kind not in KINDS:
            raise ValidationError(f"unknown model kind {self.kind!r}")
        return N.StackDesc(KINDS[self.kind], self.d, self.heads, self.ffn, self.n_enc, self.n_dec,
                           self.buffer_open, self.buffer_close, self.ln_eps, self.base_h,
                           self.dropout, self.init_std, int(self.depth_scaled_init))


@dataclass
class SolveConfig:
    """adjoint.hpp:70-79 (defaults identical)."""
    coarsen: int = 2
    levels: int = 2
    fwd_iters: int = 2
    bwd_iters: int = 1
    fwd_tol: float = 0.0
    bwd_tol: float = 0.0
    cold_guess: str = "broadcast"
    warm_start: bool = True

    def desc(self) -> N.SolveDesc:
        if self.cold_guess not in GUESSES:
            raise ValidationError(f"unknown initial guess {self.cold_guess!r}")
        return N.SolveDesc(self.coarsen, self.levels, self.fwd_iters, self.bwd_iters,
                           self.fwd_tol, self.bwd_tol, GUESSES[self.cold_guess],
                           int(self.warm_start))


@dataclass
class PhaseTrace:
    trace: List[float] = field(default_factory=list)
    converged: bool = False


@dataclass
class ForwardOutcome:
    traj: List["State"]
    phase: PhaseTrace


@dataclass
class BackwardOutcome:
    lambda0: "State"
    phase: PhaseTrace


class State:
    """One time point: encoder stream x and (encoder-decoder only) decoder stream y."""
    __slots__ = ("x", "y")

    def __init__(self, x: np.ndarray, y: Optional[np.ndarray] = None):
        self.x = np.asarray(x, np.float64)
        self.y = None if y is None else np.asarray(y, np.float64)

    @property
    def shape(self):
        b, sx, _ = self.x.shape
        return b, sx, (0 if self.y is None else self.y.shape[1])

    def flat(self) -> np.ndarray:
        parts = [self.x.ravel()] + ([] if self.y is None else [self.y.ravel()])
        return np.ascontiguousarray(np.concatenate(parts), np.float64)

    @staticmethod
    def from_flat(flat, b, sx, sy, d) -> "State":
        flat = np.asarray(flat, np.float64)
        nx = b * sx * d
        x = flat[:nx].reshape(b, sx, d).copy()
        y = flat[nx:nx + b * sy * d].reshape(b, sy, d).copy() if sy else None
        return State(x, y)

    def zeros_like(self) -> "State":
        return State(np.zeros_like(self.x), None if self.y is None else np.zeros_like(self.y))


def _open_engine(stack_cfg: StackConfig, solve_cfg: SolveConfig, device: int):
    h = C.c_void_p()
    N.call("mglp_engine_create", C.byref(stack_cfg.desc()), C.byref(solve_cfg.desc()), device,
           C.byref(h))
    return h


class _Handle:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h and N._lib is not None:
            N._lib.mglp_engine_destroy(h)
            self.h = None


class LayerStack:
    """The continuous-depth layer stack (blocks.hpp:120-175) with parameters
    initialised exactly as LayerStack(cfg, seed) does (blocks.cpp:432-449)."""

    def __init__(self, cfg: StackConfig, seed: int, device: int = 0):
        self.cfg = cfg
        self.device = device
        self._eng = _Handle(_open_engine(cfg, SolveConfig(), device))
        t, ib, ie, n = C.c_int(), C.c_int(), C.c_int(), C.c_longlong()
        N.call("mglp_engine_info", self._eng.h, C.byref(t), C.byref(ib), C.byref(ie), C.byref(n))
        self._total, self._ib, self._ie, self._np = t.value, ib.value, ie.value, n.value
        self._params = np.empty(self._np, np.float64)
        N.call("mglp_engine_init_params", self._eng.h, C.c_ulonglong(seed), N.dptr(self._params))
        self.version = 0
        self._dropout = None        # (seed, batch_index, batch, s_x, s_y) of the live masks
        self.dropout_version = 0

    # ---- accessors (blocks.hpp:124-134) ----
    def config(self):
        return self.cfg

    def total_layers(self):
        return self._total

    def interior_begin(self):
        return self._ib

    def interior_end(self):
        return self._ie

    def interior_layers(self):
        return self._ie - self._ib

    def step_size(self, layer: int) -> float:
        h = C.c_double()
        N.call("mglp_engine_step_size", self._eng.h, layer, C.byref(h))
        return h.value

    def interior_h(self):
        return self.step_size(self._ib)

    def is_buffer(self, layer):
        return layer < self.cfg.buffer_open or layer >= self._ie

    def num_params(self):
        return self._np

    def params(self) -> np.ndarray:
        """Flat parameters in visit_params order (read-only view; use set_params)."""
        v = self._params.view()
        v.flags.writeable = False
        return v

    def set_params(self, flat):
        flat = np.ascontiguousarray(flat, np.float64)
        if flat.size != self._np:
            raise ValidationError("set_params: parameter count mismatch")
        self._params = flat.copy()
        N.call("mglp_engine_set_params", self._eng.h, N.dptr(self._params), self._np)
        self.version += 1

    # ---- dropout (blocks.cpp:576-599) ----
    def refresh_dropout(self, seed: int, batch_index: int, batch: int, s_x: int, s_y: int):
        """Frozen masks of one batch for every layer (no-op if dropout <= 0)."""
        N.call("mglp_engine_refresh_dropout", self._eng.h, C.c_ulonglong(seed),
               C.c_ulonglong(batch_index), batch, s_x, s_y)
        self._dropout = (seed, batch_index, batch, s_x, s_y)
        self.dropout_version += 1

    def clear_dropout(self):
        N.call("mglp_engine_clear_dropout", self._eng.h)
        self._dropout = None
        self.dropout_version += 1

    def zero_grads(self) -> np.ndarray:
        return np.zeros(self._np, np.float64)

    # ---- Phi / Phi^T (blocks.cpp:509-574) ----
    def step(self, layer: int, dt: float, z: State) -> State:
        b, sx, sy = z.shape
        zf = z.flat()
        out = np.empty_like(zf)
        N.call("mglp_stack_step", self._eng.h, layer, dt, b, sx, sy, N.dptr(zf), N.dptr(out))
        return State.from_flat(out, b, sx, sy, self.cfg.d)

    def adjoint_step(self, layer: int, dt: float, z: State, lam: State,
                     grads: Optional[np.ndarray] = None, gscale: float = 0.0) -> State:
        b, sx, sy = z.shape
        zf, lf = z.flat(), lam.flat()
        out = np.empty_like(zf)
        N.call("mglp_stack_adjoint_step", self._eng.h, layer, dt, b, sx, sy, N.dptr(zf),
               N.dptr(lf), N.dptr(grads), gscale, N.dptr(out))
        return State.from_flat(out, b, sx, sy, self.cfg.d)


def serial_forward(stack: LayerStack, z0: State) -> List[State]:
    """blocks.cpp:659-666: the states at all total_layers()+1 time points."""
    b, sx, sy = z0.shape
    zf = z0.flat()
    traj = np.empty((stack.total_layers() + 1, zf.size), np.float64)
    N.call("mglp_serial_forward", stack._eng.h, b, sx, sy, N.dptr(zf), N.dptr(traj))
    return [State.from_flat(t, b, sx, sy, stack.cfg.d) for t in traj]


def serial_adjoint(stack: LayerStack, traj: List[State], lam_n: State,
                   grads: Optional[np.ndarray] = None) -> List[State]:
    """blocks.cpp:668-682: lambda at every time point; grads (+=) scaled by h."""
    if len(traj) != stack.total_layers() + 1:
        raise ValidationError("serial_adjoint: trajectory/stack depth mismatch")
    b, sx, sy = lam_n.shape
    tf = np.ascontiguousarray(np.stack([t.flat() for t in traj]))
    lf = lam_n.flat()
    lam = np.empty_like(tf)
    N.call("mglp_serial_adjoint", stack._eng.h, b, sx, sy, N.dptr(tf), N.dptr(lf), N.dptr(lam),
           N.dptr(grads))
    return [State.from_flat(t, b, sx, sy, stack.cfg.d) for t in lam]


@dataclass(frozen=True)
class WarmSnapshot:
    """Handle of the engine's (single) warm-state snapshot slot."""
    id: int


class LayerParallelEngine:
    """adjoint.hpp:99-219 on the device: buffers serial, the interior window
    through MGRIT forward + adjoint MGRIT, then the parameter-gradient pass."""

    def __init__(self, stack: LayerStack, cfg: SolveConfig, device: Optional[int] = None):
        self.stack = stack
        self._cfg = cfg
        self._eng = _Handle(_open_engine(stack.cfg, cfg, stack.device if device is None else device))
        self._synced = -1
        self._drop_synced = 0
        self._traj_key = None

    def _sync(self):
        if self._synced != self.stack.version or self._synced < 0:
            p = np.ascontiguousarray(self.stack._params)
            N.call("mglp_engine_set_params", self._eng.h, N.dptr(p), p.size)
            self._synced = self.stack.version
        if self._drop_synced != self.stack.dropout_version:
            # the stack's frozen masks (the reference engine reads them from the stack)
            if self.stack._dropout is not None:
                seed, k, b, sx, sy = self.stack._dropout
                N.call("mglp_engine_refresh_dropout", self._eng.h, C.c_ulonglong(seed),
                       C.c_ulonglong(k), b, sx, sy)
            else:
                N.call("mglp_engine_clear_dropout", self._eng.h)
            self._drop_synced = self.stack.dropout_version
        N.call("mglp_engine_set_config", self._eng.h, C.byref(self._cfg.desc()))

    def config(self) -> SolveConfig:
        return self._cfg

    def forward(self, z0: State, want_traj: bool = True) -> ForwardOutcome:
        self._sync()
        b, sx, sy = z0.shape
        zf = z0.flat()
        traj = np.empty((self.stack.total_layers() + 1, zf.size), np.float64) if want_traj else None
        tr = np.empty(256, np.float64)
        n, conv = C.c_int(), C.c_int()
        N.call("mglp_engine_forward", self._eng.h, b, sx, sy, N.dptr(zf), N.dptr(traj),
               N.dptr(tr), 256, C.byref(n), C.byref(conv))
        states = [] if traj is None else [State.from_flat(t, b, sx, sy, self.stack.cfg.d) for t in traj]
        self._traj_key = (id(states), b, sx, sy)
        self._last_traj = states
        return ForwardOutcome(states, PhaseTrace(list(tr[:n.value]), bool(conv.value)))

    def backward(self, traj: List[State], lam_n: State,
                 grads: Optional[np.ndarray] = None) -> BackwardOutcome:
        """grads (flat, visit_params order) are accumulated (+=), never zeroed."""
        self._sync()
        b, sx, sy = lam_n.shape
        lf = lam_n.flat()
        # reuse the device-resident trajectory when traj is the last forward's output
        tf = None
        if traj is not getattr(self, "_last_traj", None):
            if len(traj) != self.stack.total_layers() + 1:
                raise ValidationError("backward: trajectory does not match the stack depth")
            tf = np.ascontiguousarray(np.stack([t.flat() for t in traj]))
        lam0 = np.empty_like(lf)
        tr = np.empty(256, np.float64)
        n, conv = C.c_int(), C.c_int()
        N.call("mglp_engine_backward", self._eng.h, b, sx, sy, N.dptr(tf), N.dptr(lf),
               N.dptr(lam0), N.dptr(grads), N.dptr(tr), 256, C.byref(n), C.byref(conv))
        return BackwardOutcome(State.from_flat(lam0, b, sx, sy, self.stack.cfg.d),
                               PhaseTrace(list(tr[:n.value]), bool(conv.value)))

    # ---- WarmSnapshot (adjoint.hpp:187-206); one snapshot slot per engine ----
    def snapshot(self) -> "WarmSnapshot":
        sid = C.c_longlong()
        N.call("mglp_engine_snapshot_id", self._eng.h, C.byref(sid))
        return WarmSnapshot(sid.value)

    def restore(self, snap: Optional["WarmSnapshot"] = None):
        """restore(snap) raises ValidationError if `snap` is no longer the
        engine's snapshot slot (a later snapshot or a shape change replaced
        it); restore() without an argument restores the slot."""
        if snap is None:
            N.call("mglp_engine_restore", self._eng.h)
        else:
            N.call("mglp_engine_restore_id", self._eng.h, snap.id)

    def reset(self):
        N.call("mglp_engine_reset", self._eng.h)

    # ---- device-resident path (what bench.py times) ----
    @property
    def handle(self):
        return self._eng.h
