"""Gradient-bias monitor (reference include/mglp/controller.hpp:32-166).

The pure rules (last_pair_factor, decide), ProbeScope and InexactnessMonitor
keep the reference's names and semantics. DeviceMonitor evaluates the rule on
the GPU from the residual traces the solves left in device memory
(mglp_monitor_record), so no trace has to be copied to the host to decide.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List

from . import _native as N
from ._native import ValidationError

KEEP, INCREASE_ITERATIONS, SWITCH_SERIAL = 0, 1, 2
POLICY_INCREASE, POLICY_SWITCH = 0, 1
_NAMES = {KEEP: "keep", INCREASE_ITERATIONS: "increase_iterations", SWITCH_SERIAL: "switch_serial"}


def decision_name(d: int) -> str:
    return _NAMES.get(d, "?")


@dataclass
class IndicatorConfig:
    """controller.hpp:35-43."""
    probe_period: int = 500
    threshold: float = 1.0
    policy: int = POLICY_INCREASE
    max_iter_cap: int = 16
    use_probe_gradient: bool = True


@dataclass
class IndicatorReport:
    batch: int = 0
    fwd_factor: float = 0.0
    bwd_factor: float = 0.0
    decision: int = KEEP


def last_pair_factor(trace) -> float:
    """controller.hpp:63-67."""
    n = len(trace)
    if n < 2 or trace[n - 2] == 0.0:
        return 0.0
    return trace[n - 1] / trace[n - 2]


def decide(fwd_factor, bwd_factor, cfg: IndicatorConfig, fwd_iters, bwd_iters) -> int:
    """controller.hpp:71-84."""
    if cfg.threshold <= 0.0:
        raise ValidationError("decide: threshold must be positive")
    worst = max(fwd_factor, bwd_factor)
    if worst <= cfg.threshold:
        return KEEP
    if cfg.policy == POLICY_SWITCH:
        return SWITCH_SERIAL
    can_grow = fwd_iters < cfg.max_iter_cap or bwd_iters < cfg.max_iter_cap
    return INCREASE_ITERATIONS if can_grow else SWITCH_SERIAL


class ProbeScope:
    """controller.hpp:88-105: doubles both budgets for one run, then restores."""

    def __init__(self, solve_cfg):
        self.cfg = solve_cfg
        self.fwd, self.bwd = solve_cfg.fwd_iters, solve_cfg.bwd_iters

    def __enter__(self):
        self.cfg.fwd_iters = 2 * self.fwd
        self.cfg.bwd_iters = 2 * self.bwd
        return self

    def __exit__(self, *exc):
        self.cfg.fwd_iters = self.fwd
        self.cfg.bwd_iters = self.bwd
        return False


class InexactnessMonitor:
    """controller.hpp:109-155."""

    def __init__(self, cfg: IndicatorConfig):
        if cfg.probe_period < 1:
            raise ValidationError("InexactnessMonitor: probe_period must be >= 1")
        if cfg.threshold <= 0.0:
            raise ValidationError("InexactnessMonitor: threshold must be positive")
        self.cfg = cfg
        self._switched = False
        self.reports: List[IndicatorReport] = []

    def config(self):
        return self.cfg

    def switched(self) -> bool:
        return self._switched

    def due(self, batch: int) -> bool:
        return not self._switched and batch % self.cfg.probe_period == 0

    def record(self, batch, fwd_factor, bwd_factor, solve) -> IndicatorReport:
        rep = IndicatorReport(batch, fwd_factor, bwd_factor,
                              decide(fwd_factor, bwd_factor, self.cfg, solve.fwd_iters,
                                     solve.bwd_iters))
        if rep.decision == INCREASE_ITERATIONS:
            solve.fwd_iters = min(2 * solve.fwd_iters, self.cfg.max_iter_cap)
            solve.bwd_iters = min(2 * solve.bwd_iters, self.cfg.max_iter_cap)
        elif rep.decision == SWITCH_SERIAL:
            self._switched = True
        self.reports.append(rep)
        return rep


class DeviceMonitor(InexactnessMonitor):
    """InexactnessMonitor whose state lives on the GPU (mglp_*_monitor_*):
    the budgets the solves run with, the switch flag and the report log are
    device memory; record() is one kernel evaluating last_pair_factor on the
    device-resident traces, decide() and the budget update. The host keeps a
    mirror of `switched` (refreshed by every probe) for due(); reports()
    copies the device log."""

    def __init__(self, cfg: IndicatorConfig, handle, trainer: bool):
        super().__init__(cfg)
        self._h = handle
        self._trainer = trainer
        pre = "mglp_trainer" if trainer else "mglp_engine"
        N.call(pre + "_monitor_attach", handle, cfg.threshold,
               int(cfg.policy == POLICY_SWITCH), cfg.max_iter_cap)

    def record_engine(self, batch) -> IndicatorReport:
        """engine users: record() after engine.forward/backward"""
        dec, sw = C.c_int(), C.c_int()
        ff, bf = C.c_double(), C.c_double()
        N.call("mglp_monitor_record", self._h, batch, None)
        N.call("mglp_engine_monitor_read", self._h, C.byref(sw), C.byref(dec), C.byref(ff),
               C.byref(bf), None, None, None, None)
        self._switched = bool(sw.value)
        return IndicatorReport(batch, ff.value, bf.value, dec.value)

    def note(self, switched: bool):
        self._switched = bool(switched)

    @property
    def reports(self) -> List[IndicatorReport]:
        cap = 1024
        b = (C.c_longlong * cap)()
        ff, bf = (C.c_double * cap)(), (C.c_double * cap)()
        dec = (C.c_int * cap)()
        n = C.c_int()
        pre = "mglp_trainer" if self._trainer else "mglp_engine"
        N.call(pre + "_monitor_reports", self._h, b, ff, bf, dec, cap, C.byref(n))
        return [IndicatorReport(b[i], ff[i], bf[i], dec[i]) for i in range(min(n.value, cap))]

    @reports.setter
    def reports(self, v):  # InexactnessMonitor.__init__ assigns []
        pass


def indicator_csv(reports) -> str:
    """controller.hpp:157-166."""
    out = "batch, fwd_factor, bwd_factor, decision\n"
    for r in reports:
        out += f"{r.batch}, {r.fwd_factor:.17g}, {r.bwd_factor:.17g}, {decision_name(r.decision)}\n"
    return out
