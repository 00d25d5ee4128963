"""Lipschitz probe and buffer-layer selection: the reference's lipschitz.hpp
API (lipschitz.cpp:53-277), with the probe itself on the device.

`estimate_stack` / `estimate_lipschitz` run every layer's residual map F on
the GPU (probe.cu: all samples of a layer as one batch, the reference's
counter-based draws regenerated on the device); the buffer selection,
recommendation, weight-drift tracking and CSV tables are host logic restated
from lipschitz.cpp with the same rules and messages.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple, Union

import numpy as np

from . import _native as N
from ._native import ContractViolation, ValidationError

kUndefinedChange = -1.0  # lipschitz.hpp: rel_change when the snapshot norm is zero


@dataclass
class ProbeConfig:  # lipschitz.hpp ProbeConfig
    samples: int = 1000
    delta_scale: float = 1e-2   # perturbation magnitude per element
    input_scale: float = 1.0    # base-point scale; match activation RMS
    seq_len: int = 8            # sequence length of probe inputs


@dataclass
class LipschitzEstimate:  # lipschitz.hpp LipschitzEstimate
    layer: int = 0
    estimate: float = 0.0
    samples: int = 0
    input_scale: float = 1.0
    delta_scale: float = 0.0
    seed: int = 0


def _probe(stack, layers: Sequence[int], cfg: ProbeConfig, seed: int) -> List[LipschitzEstimate]:
    if cfg.samples < 1:
        raise ValidationError("estimate_lipschitz: need at least one sample")
    arr = (C.c_int * len(layers))(*layers)
    out = np.zeros(len(layers), np.float64)
    N.call("mglp_engine_lipschitz", stack._eng.h, int(cfg.samples), float(cfg.delta_scale),
           float(cfg.input_scale), int(cfg.seq_len), C.c_ulonglong(seed), arr, len(layers),
           N.dptr(out))
    return [LipschitzEstimate(layer=int(l), estimate=float(e), samples=cfg.samples,
                              input_scale=cfg.input_scale, delta_scale=cfg.delta_scale, seed=seed)
            for l, e in zip(layers, out)]


def estimate_lipschitz(stack, layer: int, cfg: ProbeConfig, seed: int) -> LipschitzEstimate:
    """lipschitz.cpp:90-139: max over cfg.samples draws of ||F(x+d) - F(x)|| / ||d||
    for the residual map F of one layer (cross-attention layers against a
    frozen context)."""
    if layer < 0 or layer >= stack.total_layers():
        raise ValidationError("estimate_lipschitz: layer out of range")
    return _probe(stack, [layer], cfg, seed)[0]


def estimate_stack(stack, cfg: ProbeConfig, seed: int) -> List[LipschitzEstimate]:
    """lipschitz.cpp:141-149: every layer, in order (one device call)."""
    return _probe(stack, list(range(stack.total_layers())), cfg, seed)


@dataclass
class BufferPlan:  # lipschitz.hpp BufferPlan
    k_open: int = 0
    k_close: int = 0
    buffered: List[int] = field(default_factory=list)
    interior_spike: bool = False
    warning: str = ""


def select_buffer_layers(estimates: Sequence[LipschitzEstimate], k_open: int,
                         k_close: int) -> BufferPlan:
    """lipschitz.cpp:151-184: flag the k_open first / k_close last layers and
    warn when an interior estimate tops every buffered one."""
    n = len(estimates)
    if k_open < 0 or k_close < 0:
        raise ValidationError("select_buffer_layers: negative buffer count")
    if k_open + k_close >= n:
        raise ValidationError("select_buffer_layers: buffers would swallow the stack")
    plan = BufferPlan(k_open=k_open, k_close=k_close)
    plan.buffered = [estimates[i].layer for i in range(k_open)] + \
        [estimates[i].layer for i in range(n - k_close, n)]
    if plan.buffered:
        max_buffered = 0.0
        for i in list(range(k_open)) + list(range(n - k_close, n)):
            max_buffered = max(max_buffered, estimates[i].estimate)
        for i in range(k_open, n - k_close):
            if estimates[i].estimate > max_buffered:
                plan.interior_spike = True
                plan.warning = (f"layer {estimates[i].layer} estimate {_g6(estimates[i].estimate)} "
                                f"exceeds every buffered layer (max {_g6(max_buffered)}); "
                                f"buffers may be misplaced")
                break
    return plan


@dataclass
class BufferRecommendation:  # lipschitz.hpp BufferRecommendation
    k_open: int = 0
    k_close: int = 0
    amp_threshold: float = 2.0


def recommend_buffers(amplification: Union[Sequence[float], Sequence[LipschitzEstimate]],
                      stack=None, amp_threshold: float = 2.0) -> BufferRecommendation:
    """lipschitz.cpp:219-251: the hot end runs (amplification 1 + h L >=
    threshold) become buffers, always leaving an interior window. Pass
    estimates + stack to use each layer's own step size."""
    if stack is not None:
        amps = [1.0 + stack.step_size(e.layer) * e.estimate for e in amplification]
    else:
        amps = [float(a) for a in amplification]
    if amp_threshold <= 1.0:
        raise ValidationError("recommend_buffers: threshold must exceed 1")
    n = len(amps)
    rec = BufferRecommendation(amp_threshold=amp_threshold)
    while rec.k_open < n and amps[rec.k_open] >= amp_threshold:
        rec.k_open += 1
    while rec.k_close < n and amps[n - 1 - rec.k_close] >= amp_threshold:
        rec.k_close += 1
    # a fully hot stack still needs an interior window to parallelize
    while n > 0 and rec.k_open + rec.k_close >= n:
        if rec.k_close >= rec.k_open and rec.k_close > 0:
            rec.k_close -= 1
        else:
            rec.k_open -= 1
    return rec


def _g6(x: float) -> str:
    return f"{x:.6g}"


def _g17(x: float) -> str:
    return f"{x:.17g}"


def lipschitz_csv(estimates: Sequence[LipschitzEstimate], stack) -> str:
    """lipschitz.cpp:253-265: per layer estimate and amplification 1 + h L."""
    out = "layer, estimate, amplification, samples, seed\n"
    for e in estimates:
        amp = 1.0 + stack.step_size(e.layer) * e.estimate
        out += f"{e.layer}, {_g17(e.estimate)}, {_g17(amp)}, {e.samples}, {e.seed}\n"
    return out


def param_layout(cfg) -> List[Tuple[int, str, int, int]]:
    """(layer, component, offset, size) of every tensor in visit_params order
    (blocks.cpp:604-646) for a StackConfig."""
    d, f = cfg.d, cfg.ffn
    kind = cfg.kind
    total = cfg.n_enc + cfg.n_dec if kind == "encoder_decoder" else \
        (cfg.n_enc if kind == "encoder" else cfg.n_dec)
    out, off = [], 0

    def add(layer, name, n):
        nonlocal off
        out.append((layer, name, off, n))
        off += n

    def lin(layer, p, o, i):
        add(layer, p + ".w", o * i)
        add(layer, p + ".b", o)

    def ln(layer, p):
        add(layer, p + ".gain", d)
        add(layer, p + ".bias", d)

    def attn(layer, p):
        for s in ("q", "k", "v", "o"):
            lin(layer, f"{p}.{s}", d, d)

    for layer in range(total):
        if kind == "encoder_decoder" and layer >= cfg.n_enc:
            ln(layer, "ln1")
            attn(layer, "self")
            ln(layer, "ln3")
            attn(layer, "cross")
        else:
            ln(layer, "ln1")
            attn(layer, "attn")
        ln(layer, "ln2")
        lin(layer, "mlp.in", f, d)
        lin(layer, "mlp.out", d, f)
    return out


@dataclass
class WeightChange:  # lipschitz.hpp WeightChange
    layer: int = 0
    component: str = ""
    rel_change: float = 0.0


def track_weight_change(now: np.ndarray, base: np.ndarray, cfg) -> List[WeightChange]:
    """lipschitz.cpp:186-217: per tensor ||now - base|| / ||base|| (0 for no
    drift; kUndefinedChange for drift away from a zero snapshot). `now` and
    `base` are flat parameter vectors in visit_params order."""
    now = np.asarray(now, np.float64)
    base = np.asarray(base, np.float64)
    layout = param_layout(cfg)
    total = sum(n for _, _, _, n in layout)
    if now.size != total or base.size != total:
        raise ContractViolation("track_weight_change: parameter sets do not line up")
    out = []
    for layer, comp, off, n in layout:
        a, b = now[off:off + n], base[off:off + n]
        base_norm = math.sqrt(_seq_sumsq(b))
        drift = math.sqrt(_seq_sumsq(a - b))
        if drift == 0.0:
            rel = 0.0
        else:
            rel = drift / base_norm if base_norm > 0.0 else kUndefinedChange
        out.append(WeightChange(layer=layer, component=comp, rel_change=rel))
    return out


def _seq_sumsq(v: np.ndarray) -> float:
    """sum of squares accumulated in element order (lipschitz.cpp:29-42)"""
    return float(np.cumsum(v * v)[-1]) if v.size else 0.0


def weight_change_csv(changes: Sequence[WeightChange]) -> str:
    """lipschitz.cpp:267-275"""
    out = "layer, component, rel_change\n"
    for c in changes:
        out += f"{c.layer}, {c.component}, {_g17(c.rel_change)}\n"
    return out
