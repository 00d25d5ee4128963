"""Training loop around the device engine: the reference's Trainer
(training.cpp:69-318) with its per-batch update on the B200.

The per-batch work (Trainer::run_update, training.cpp:230-268 -- batch
generation, embedding, the layer-parallel or serial solve, logits /
cross-entropy / head backward, embedding backward and the optimizer step)
runs on the device behind the C-ABI (mglp_trainer_*, csrc/trainer.cu). This
module keeps the host-side schedule of the reference: the mode switch,
monitor probes (ProbeScope doubling, snapshot/restore), validation cadence,
metrics CSV, config echo and the MGLP v1 handover / final checkpoints.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N
from ._native import ValidationError
from .controller import (INCREASE_ITERATIONS, SWITCH_SERIAL, DeviceMonitor, IndicatorConfig,
                         IndicatorReport,
                         InexactnessMonitor, ProbeScope, last_pair_factor)
from .engine import KINDS, SolveConfig, StackConfig

TASKS = {"copy_sequence": 0, "token_classification": 1, "tiny_translation": 2}
OPTS = {"sgd": 0, "adam": 1, "adamw": 2}
MODES = ("serial", "layer_parallel", "switching")


@dataclass
class TaskSpec:
    """tasks.hpp:24-42."""
    kind: str = "copy_sequence"
    vocab: int = 16
    seq_len: int = 8
    train_size: int = 256
    val_size: int = 64
    seed: int = 1

    def desc(self) -> N.TaskDesc:
        if self.kind not in TASKS:
            raise ValidationError(f"unknown task {self.kind!r}")
        return N.TaskDesc(TASKS[self.kind], self.vocab, self.seq_len, self.train_size,
                          self.val_size, self.seed)


@dataclass
class ModelConfig:
    """model.hpp:32-36."""
    stack: StackConfig = field(default_factory=StackConfig)
    vocab: int = 16
    max_seq: int = 16


@dataclass
class OptConfig:
    """optimizer.hpp:26-34."""
    kind: str = "adamw"
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01
    momentum: float = 0.0

    def desc(self) -> N.OptDesc:
        if self.kind not in OPTS:
            raise ValidationError(f"unknown optimizer {self.kind!r}")
        return N.OptDesc(OPTS[self.kind], self.lr, self.beta1, self.beta2, self.eps,
                         self.weight_decay, self.momentum)


@dataclass
class TrainConfig:
    """training.hpp:33-46."""
    mode: str = "layer_parallel"
    opt: OptConfig = field(default_factory=OptConfig)
    solve: SolveConfig = field(default_factory=SolveConfig)
    indicator: IndicatorConfig = field(default_factory=IndicatorConfig)
    batch_size: int = 8
    epochs: int = 1
    workers: int = 1
    seed: int = 7
    manual_switch_batch: int = -1
    val_every: int = 25


@dataclass
class MetricsRow:
    """training.hpp:48-57."""
    batch: int = 0
    loss: float = 0.0
    val_metric: float = 0.0
    mode: str = ""
    fwd_iters: int = 0
    bwd_iters: int = 0
    fwd_factor: float = 0.0
    bwd_factor: float = 0.0


@dataclass
class TrainResult:
    """training.hpp:59-68."""
    rows: List[MetricsRow] = field(default_factory=list)
    reports: List[IndicatorReport] = field(default_factory=list)
    switched: bool = False
    switch_batch: int = -1
    final_val: float = 0.0
    csv: str = ""
    switch_state: bytes = b""
    final_state: bytes = b""


def _g17(x: float) -> str:
    return "%.17g" % x


def metrics_csv(rows: List[MetricsRow]) -> str:
    """training.cpp:315-327."""
    out = ("batch, loss, val_metric, mode, fwd_iters, bwd_iters, fwd_factor, "
           "bwd_factor\n")
    for r in rows:
        out += (f"{r.batch}, {_g17(r.loss)}, {_g17(r.val_metric)}, {r.mode}, {r.fwd_iters}, "
                f"{r.bwd_iters}, {_g17(r.fwd_factor)}, {_g17(r.bwd_factor)}\n")
    return out


def config_echo(task: TaskSpec, mcfg: ModelConfig, tcfg: TrainConfig) -> str:
    """training.cpp:329-346 (byte-identical)."""
    s = mcfg.stack
    return (f"task={task.kind} vocab={task.vocab} seq={task.seq_len} train={task.train_size} "
            f"val={task.val_size} data_seed={task.seed} | kind={s.kind} d={s.d} "
            f"heads={s.heads} ffn={s.ffn} enc={s.n_enc} dec={s.n_dec} open={s.buffer_open} "
            f"close={s.buffer_close} dropout={_g17(s.dropout)} | opt={tcfg.opt.kind} "
            f"lr={_g17(tcfg.opt.lr)} wd={_g17(tcfg.opt.weight_decay)} | "
            f"coarsen={tcfg.solve.coarsen} levels={tcfg.solve.levels} | "
            f"batch={tcfg.batch_size} epochs={tcfg.epochs} seed={tcfg.seed}")


class _EngineBudget:
    """engine_->config() seen by ProbeScope / InexactnessMonitor: reads and
    writes the device engine's iteration budget."""

    def __init__(self, h):
        self._h = h

    def _get(self):
        f, b = C.c_int(), C.c_int()
        N.call("mglp_trainer_get_iters", self._h, C.byref(f), C.byref(b))
        return f.value, b.value

    @property
    def fwd_iters(self):
        return self._get()[0]

    @fwd_iters.setter
    def fwd_iters(self, v):
        N.call("mglp_trainer_set_iters", self._h, int(v), self._get()[1])

    @property
    def bwd_iters(self):
        return self._get()[1]

    @bwd_iters.setter
    def bwd_iters(self, v):
        N.call("mglp_trainer_set_iters", self._h, self._get()[0], int(v))


class DeviceTrainer:
    """The per-batch device step (mglp_trainer_*): Model + Optimizer + engine."""

    def __init__(self, task: TaskSpec, mcfg: ModelConfig, tcfg: TrainConfig, device: int = 0):
        self.task, self.mcfg, self.tcfg = task, mcfg, tcfg
        h = C.c_void_p()
        N.call("mglp_trainer_create", C.byref(mcfg.stack.desc()), C.byref(tcfg.solve.desc()),
               C.byref(task.desc()), C.byref(tcfg.opt.desc()), mcfg.vocab, mcfg.max_seq,
               tcfg.batch_size, tcfg.seed, device, C.byref(h))
        self.h = h
        n = C.c_longlong()
        N.call("mglp_trainer_num_params", h, C.byref(n))
        self.n_params = n.value
        self.budget = _EngineBudget(h)

    def __del__(self):
        h = getattr(self, "h", None)
        if h and N._lib is not None:
            N._lib.mglp_trainer_destroy(h)
            self.h = None

    def update(self, k: int, parallel: bool, apply: bool = True) -> float:
        loss = C.c_double()
        N.call("mglp_trainer_update", self.h, k, int(parallel), int(apply), C.byref(loss))
        return loss.value

    def evaluate(self) -> float:
        acc = C.c_double()
        N.call("mglp_trainer_evaluate", self.h, C.byref(acc))
        return acc.value

    def trace(self, fwd: bool) -> List[float]:
        buf = (C.c_double * 256)()
        n, conv = C.c_int(), C.c_int()
        N.call("mglp_trainer_trace", self.h, int(fwd), buf, 256, C.byref(n), C.byref(conv))
        return list(buf[: min(n.value, 256)])

    def params(self) -> np.ndarray:
        out = np.zeros(self.n_params)
        N.call("mglp_trainer_get_params", self.h, N.dptr(out))
        return out

    def set_params(self, flat: np.ndarray):
        flat = np.ascontiguousarray(flat, dtype=np.float64)
        if flat.size != self.n_params:
            raise ValidationError("set_params: wrong parameter count")
        N.call("mglp_trainer_set_params", self.h, N.dptr(flat))

    def grads(self) -> np.ndarray:
        out = np.zeros(self.n_params)
        N.call("mglp_trainer_get_grads", self.h, N.dptr(out))
        return out

    def logits(self) -> np.ndarray:
        B, S, V = self.tcfg.batch_size, self.task.seq_len, self.mcfg.vocab
        out = np.zeros((B * S, V), dtype=np.float32)
        N.call("mglp_trainer_read_logits", self.h, out.ctypes.data_as(C.POINTER(C.c_float)))
        return out.reshape(B, S, V)

    def read_batch(self, split: int, start: int):
        """device make_batch -> (src, tgt_in, tgt_out) int32 arrays [B*seq]"""
        n = self.tcfg.batch_size * self.task.seq_len
        src, tin, tout = (np.zeros(n, dtype=np.int32) for _ in range(3))
        ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
        N.call("mglp_trainer_read_batch", self.h, split, start, ip(src), ip(tin), ip(tout))
        return src, tin, tout

    def snapshot(self):
        N.call("mglp_trainer_snapshot", self.h)

    def restore(self):
        N.call("mglp_trainer_restore", self.h)

    def save_checkpoint(self, batch: int, echo: str) -> bytes:
        e = echo.encode()
        n = C.c_longlong()
        N.call("mglp_trainer_save_checkpoint", self.h, batch, e, len(e), None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value)
        N.call("mglp_trainer_save_checkpoint", self.h, batch, e, len(e), buf, n.value,
               C.byref(n))
        return buf.raw[: n.value]

    def load_checkpoint(self, blob: bytes):
        """-> (batch, config_echo, has_optimizer)"""
        batch, elen, has = C.c_longlong(), C.c_longlong(), C.c_int()
        echo = C.create_string_buffer(4096)
        N.call("mglp_trainer_load_checkpoint", self.h, blob, len(blob), C.byref(batch), echo,
               4096, C.byref(elen), C.byref(has))
        return batch.value, echo.raw[: elen.value].decode(), bool(has.value)


class Trainer:
    """training.cpp:69-312 with the device step."""

    def __init__(self, task: TaskSpec, mcfg: ModelConfig, tcfg: TrainConfig, device: int = 0):
        self._validate(task, mcfg, tcfg)
        self.task, self.mcfg, self.tcfg = task, mcfg, tcfg
        self.dev = DeviceTrainer(task, mcfg, tcfg, device)
        # the switching mode's monitor runs on the device (DeviceMonitor):
        # budgets, decisions, switch flag and report log in GPU memory
        self.mon = (DeviceMonitor(tcfg.indicator, self.dev.h, trainer=True)
                    if tcfg.mode == "switching" else InexactnessMonitor(tcfg.indicator))
        self.batches_per_epoch = task.train_size // tcfg.batch_size
        self.total_batches = tcfg.epochs * self.batches_per_epoch
        self.echo = config_echo(task, mcfg, tcfg)

    @staticmethod
    def _validate(task, mcfg, tcfg):  # training.cpp:180-206
        if tcfg.batch_size < 1:
            raise ValidationError("train: batch_size must be >= 1")
        if tcfg.epochs < 1:
            raise ValidationError("train: epochs must be >= 1")
        if tcfg.val_every < 1:
            raise ValidationError("train: val_every must be >= 1")
        if tcfg.workers < 1:
            raise ValidationError("train: workers must be >= 1")
        if tcfg.mode not in MODES:
            raise ValidationError(f"train: unknown mode {tcfg.mode!r}")
        if task.vocab != mcfg.vocab:
            raise ValidationError("train: task and model vocabularies differ")
        if task.seq_len > mcfg.max_seq:
            raise ValidationError("train: sequence longer than the position table")
        if (task.kind == "tiny_translation") != (mcfg.stack.kind == "encoder_decoder"):
            raise ValidationError(
                "train: translation needs an encoder-decoder model, and only translation feeds one")
        if task.train_size % tcfg.batch_size != 0 or task.val_size % tcfg.batch_size != 0:
            raise ValidationError("train: split sizes must be divisible by batch_size")

    def _update(self, k, parallel, ftr=None, btr=None, apply=True) -> float:
        loss = self.dev.update(k, parallel, apply)
        if parallel:
            if ftr is not None:
                ftr[:] = self.dev.trace(True)
            if btr is not None:
                btr[:] = self.dev.trace(False)
        return loss

    def _probe_batch(self, k, row: MetricsRow):  # training.cpp:244-276
        """ProbeScope, the update and record() run on the device
        (mglp_trainer_update_probe); one synchronisation for the whole row."""
        loss = C.c_double()
        fi, bi, dec, sw = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        ff, bf = C.c_double(), C.c_double()
        N.call("mglp_trainer_update_probe", self.dev.h, k,
               int(self.tcfg.indicator.use_probe_gradient), C.byref(loss), C.byref(fi),
               C.byref(bi), C.byref(ff), C.byref(bf), C.byref(dec), C.byref(sw))
        row.loss = loss.value
        row.fwd_iters, row.bwd_iters = fi.value, bi.value
        row.fwd_factor, row.bwd_factor = ff.value, bf.value
        self.mon.note(sw.value)

    def capture(self, next_batch: int) -> bytes:
        return self.dev.save_checkpoint(next_batch, self.echo)

    def run(self) -> TrainResult:  # training.cpp:92-135
        res = TrainResult()
        serial_now = self.tcfg.mode == "serial"
        monitored = self.tcfg.mode == "switching"
        val, have_val = 0.0, False
        for k in range(self.total_batches):
            if (not serial_now and self.tcfg.manual_switch_batch >= 0
                    and k == self.tcfg.manual_switch_batch):
                res.switch_state = self.capture(k)
                res.switched, res.switch_batch = True, k
                serial_now = True
            row = MetricsRow(batch=k, mode="serial" if serial_now else "layer_parallel")
            if serial_now:
                row.loss = self._update(k, False)
            elif monitored and self.mon.due(k):
                self._probe_batch(k, row)
                if self.mon.switched() and not res.switched:
                    res.switch_state = self.capture(k + 1)
                    res.switched, res.switch_batch = True, k + 1
                    serial_now = True
            elif monitored:
                # factors of this update's traces, evaluated on the device
                row.loss = self._update(k, True)
                ff, bf, fi, bi = C.c_double(), C.c_double(), C.c_int(), C.c_int()
                N.call("mglp_trainer_last_factors", self.dev.h, C.byref(ff), C.byref(bf),
                       C.byref(fi), C.byref(bi))
                row.fwd_iters, row.bwd_iters = fi.value, bi.value
                row.fwd_factor, row.bwd_factor = ff.value, bf.value
            else:
                ftr, btr = [], []
                row.fwd_iters = self.dev.budget.fwd_iters
                row.bwd_iters = self.dev.budget.bwd_iters
                row.loss = self._update(k, True, ftr, btr, True)
                row.fwd_factor = last_pair_factor(ftr)
                row.bwd_factor = last_pair_factor(btr)
            if not have_val or k % self.tcfg.val_every == 0 or k == self.total_batches - 1:
                val = self.dev.evaluate()
                have_val = True
            row.val_metric = val
            res.rows.append(row)
        res.reports = list(self.mon.reports)
        res.final_val = val
        res.csv = metrics_csv(res.rows)
        res.final_state = self.capture(self.total_batches)
        return res

    def resume_serial(self, blob: bytes) -> TrainResult:  # training.cpp:138-154
        batch, echo, _ = self.dev.load_checkpoint(blob)
        if echo != self.echo:
            raise ValidationError("resume: checkpoint belongs to a different run")
        res = TrainResult()
        for k in range(batch, self.total_batches):
            res.rows.append(MetricsRow(batch=k, mode="serial", loss=self._update(k, False)))
        res.final_state = self.capture(self.total_batches)
        return res

    def load_start(self, blob: bytes):  # training.cpp:157-165
        batch, echo, _ = self.dev.load_checkpoint(blob)
        if echo != self.echo:
            raise ValidationError("train: start checkpoint belongs to a different run")
        if batch != 0:
            raise ValidationError("train: start checkpoint is mid-run; resume instead")


def run_training(task: TaskSpec, mcfg: ModelConfig, tcfg: TrainConfig,
                 start_state: Optional[bytes] = None, device: int = 0) -> TrainResult:
    """training.cpp:348-360."""
    t = Trainer(task, mcfg, tcfg, device)
    if start_state:
        t.load_start(start_state)
    return t.run()


@dataclass
class ReplayOutcome:
    switched: bool = False
    switch_batch: int = -1
    compared_batches: int = 0
    losses_match: bool = False
    state_matches: bool = False


def switching_replay(task, mcfg, tcfg, start_state: Optional[bytes] = None,
                     device: int = 0) -> ReplayOutcome:
    """training.cpp:362-396: re-run the post-switch tail from the captured
    handover checkpoint on the serial path; losses and final state must agree
    bitwise (the device step is deterministic)."""
    first = run_training(task, mcfg, tcfg, start_state, device)
    out = ReplayOutcome(switched=first.switched, switch_batch=first.switch_batch)
    if not first.switched:
        return out
    tail = Trainer(task, mcfg, tcfg, device)
    second = tail.resume_serial(first.switch_state)
    out.compared_batches = len(second.rows)
    out.losses_match = all(
        r.batch < len(first.rows) and
        np.float64(first.rows[r.batch].loss).tobytes() == np.float64(r.loss).tobytes()
        for r in second.rows)
    out.state_matches = first.final_state == second.final_state
    return out


# ---- MGLP v1 container (checkpoint.cpp:30-180), host-side reader ----------------
def parse_checkpoint(blob: bytes):
    """-> dict(version, config_echo, batch, params [arrays], has_optimizer,
    steps, m [arrays], v [arrays])"""
    import struct
    pos = 0

    def take(n):
        nonlocal pos
        if pos + n > len(blob):
            raise ValidationError("checkpoint: truncated stream")
        b = blob[pos:pos + n]
        pos += n
        return b

    if take(4) != b"MGLP":
        raise ValidationError("checkpoint: bad magic")
    u32 = lambda: struct.unpack("<I", take(4))[0]  # noqa: E731
    u64 = lambda: struct.unpack("<Q", take(8))[0]  # noqa: E731
    out = {"version": u32()}
    out["config_echo"] = take(u64()).decode()
    out["batch"] = u64()

    def tensors():
        ts = []
        for _ in range(u32()):
            rank = u32()
            shape = [u64() for _ in range(rank)]
            n = int(np.prod(shape)) if shape else 1
            ts.append(np.frombuffer(take(8 * n), dtype="<f8").reshape(shape).copy())
        return ts

    out["params"] = tensors()
    out["has_optimizer"] = take(1) != b"\x00"
    if out["has_optimizer"]:
        out["steps"] = u64()
        out["m"] = tensors()
        out["v"] = tensors()
    return out
