"""TEST INFRASTRUCTURE: float64 numpy restatement ("port") of the reference hot path.

This is the oracle the CUDA path is checked against when the compiled
reference (oracle/_ref, see oracle/ref.py) is not available, and it is itself
pinned against that compiled reference and the committed golden fixtures in
tests/test_oracle.py. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import it; the product path never does.

Everything follows /root/reference/proj (citations are path:line there):
  tensor primitives      src/tensor.cpp:205-372
  attention + VJP        src/blocks.cpp:142-236
  block residuals + VJPs src/blocks.cpp:246-333
  LayerStack             src/blocks.cpp:385-574, include/mglp/blocks.hpp:120-175
  serial sweeps          src/blocks.cpp:659-682
  MgritSolver            include/mglp/mgrit.hpp:58-303
  Stack{Forward,Adjoint}System  include/mglp/systems.hpp:80-102, adjoint.hpp:35-65
  LayerParallelEngine    include/mglp/adjoint.hpp:99-219
  controller             include/mglp/controller.hpp:63-155
Batched numpy contractions reassociate the reference's ascending-k sums, so
agreement with the compiled reference is ~1e-13 relative, not bitwise.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

KMASK = -1e30  # blocks.cpp:85
GELU_C = 0.7978845608028654  # tensor.cpp:345
GELU_A = 0.044715  # tensor.cpp:346

# ---------------------------------------------------------------------------
# parameters (visit_params order, blocks.cpp:627-646)
# ---------------------------------------------------------------------------

ENC_FIELDS = ["ln1", "attn", "ln2", "mlp.in", "mlp.out"]


def layer_components(is_decoder: bool, d: int, ffn: int):
    """(name, shape) in visit_params order for one block."""
    def lin(prefix, out, inp):
        return [(prefix + ".w", (out, inp)), (prefix + ".b", (out,))]

    def ln(prefix):
        return [(prefix + ".gain", (d,)), (prefix + ".bias", (d,))]

    def attn(prefix):
        return sum((lin(f"{prefix}.{k}", d, d) for k in "qkvo"), [])

    if not is_decoder:
        return ln("ln1") + attn("attn") + ln("ln2") + lin("mlp.in", ffn, d) + lin("mlp.out", d, ffn)
    return (ln("ln1") + attn("self") + ln("ln3") + attn("cross") + ln("ln2")
            + lin("mlp.in", ffn, d) + lin("mlp.out", d, ffn))


@dataclass
class StackConfig:
    kind: str = "encoder"  # encoder | decoder_only | encoder_decoder
    d: int = 32
    heads: int = 2
    ffn: int = 64
    n_enc: int = 8
    n_dec: int = 0
    buffer_open: int = 0
    buffer_close: int = 0
    ln_eps: float = 1e-5
    base_h: float = 1.0


class Stack:
    """LayerStack restated (blocks.cpp:385-450 for shape/h; params come in flat)."""

    def __init__(self, cfg: StackConfig, flat_params: np.ndarray):
        self.cfg = cfg
        if cfg.kind == "encoder":
            total, self.n_split = cfg.n_enc, cfg.n_enc
        elif cfg.kind == "decoder_only":
            total, self.n_split = cfg.n_dec, cfg.n_dec
        else:
            total, self.n_split = cfg.n_enc + cfg.n_dec, cfg.n_enc
        self.total = total
        self.causal = cfg.kind == "decoder_only"
        self.ib = cfg.buffer_open
        self.ie = total - cfg.buffer_close
        self.h = [cfg.base_h] * total  # blocks.cpp:421-430
        if cfg.buffer_open + cfg.buffer_close > 0:
            interior = total - cfg.buffer_open - cfg.buffer_close
            for i in range(total):
                buf = i < cfg.buffer_open or i >= total - cfg.buffer_close
                self.h[i] = 1.0 if buf else 1.0 / interior
        self.params = self.unflatten(flat_params)

    def is_decoder(self, layer):
        return self.cfg.kind == "encoder_decoder" and layer >= self.n_split

    def unflatten(self, flat):
        flat = np.asarray(flat, np.float64)
        out, o = [], 0
        for layer in range(self.total):
            p = {}
            for name, shp in layer_components(self.is_decoder(layer), self.cfg.d, self.cfg.ffn):
                n = int(np.prod(shp))
                p[name] = flat[o:o + n].reshape(shp)
                o += n
            out.append(p)
        assert o == flat.size, (o, flat.size)
        return out

    def zero_grads(self):
        return [{k: np.zeros_like(v) for k, v in p.items()} for p in self.params]

    @staticmethod
    def flatten(blocks):
        return np.concatenate([v.ravel() for p in blocks for v in p.values()])

    @property
    def interior_layers(self):
        return self.ie - self.ib

    def interior_h(self):
        return self.h[self.ib]

    # ---- F and its VJP (blocks.cpp:466-564) ----
    def residual(self, layer, z):
        p = self.params[layer]
        H, eps = self.cfg.heads, self.cfg.ln_eps
        if layer < self.n_split:
            fx = encoder_residual(p, H, self.causal, eps, z.x)
            return State(fx, None if z.y is None else np.zeros_like(z.y))
        fy = decoder_residual(p, H, eps, z.y, z.x)
        return State(np.zeros_like(z.x), fy)

    def step(self, layer, dt, z):
        f = self.residual(layer, z)
        return z.axpy(dt, f)

    def residual_vjp(self, layer, z, lam, grads, gscale):
        p = self.params[layer]
        H, eps = self.cfg.heads, self.cfg.ln_eps
        g = grads[layer] if grads is not None else None
        if layer < self.n_split:
            rx = encoder_residual_vjp(p, H, self.causal, eps, z.x, lam.x, g, gscale)
            return State(rx, None if z.y is None else np.zeros_like(z.y))
        dy, dxe = decoder_residual_vjp(p, H, eps, z.y, z.x, lam.y, g, gscale)
        return State(dxe, dy)

    def adjoint_step(self, layer, dt, z, lam, grads, gscale):
        r = self.residual_vjp(layer, z, lam, grads, gscale)
        return lam.axpy(dt, r)


# ---------------------------------------------------------------------------
# State algebra (blocks.cpp:25-79)
# ---------------------------------------------------------------------------


class State:
    __slots__ = ("x", "y")

    def __init__(self, x, y=None):
        self.x = x
        self.y = y

    def _map2(self, o, f):
        return State(None if self.x is None else f(self.x, o.x),
                     None if self.y is None else f(self.y, o.y))

    def __add__(self, o):
        return self._map2(o, lambda a, b: a + b)

    def __sub__(self, o):
        return self._map2(o, lambda a, b: a - b)

    def axpy(self, c, o):
        # a + c*b, the reference's axpy (tensor.cpp:105-110): a[i] += s*b[i]
        return self._map2(o, lambda a, b: a + c * b)

    def copy(self):
        return State(None if self.x is None else self.x.copy(),
                     None if self.y is None else self.y.copy())

    def zeros_like(self):
        return State(None if self.x is None else np.zeros_like(self.x),
                     None if self.y is None else np.zeros_like(self.y))

    def norm_sq(self):
        s = 0.0
        if self.x is not None:
            s += float(np.dot(self.x.ravel(), self.x.ravel()))
        if self.y is not None:
            s += float(np.dot(self.y.ravel(), self.y.ravel()))
        return s

    def flat(self):
        parts = [a.ravel() for a in (self.x, self.y) if a is not None]
        return np.concatenate(parts)

    @staticmethod
    def from_flat(flat, b, sx, sy, d):
        flat = np.asarray(flat, np.float64)
        nx = b * sx * d
        x = flat[:nx].reshape(b, sx, d).copy() if sx else None
        y = flat[nx:nx + b * sy * d].reshape(b, sy, d).copy() if sy else None
        return State(x, y)


# ---------------------------------------------------------------------------
# primitives (tensor.cpp)
# ---------------------------------------------------------------------------


def linear(x, w, b):
    return x @ w.T + b


def layer_norm(x, gain, bias, eps):
    mean = x.mean(-1, keepdims=True)
    c = x - mean
    var = (c * c).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    return gain * (c * rstd) + bias


def layer_norm_vjp(x, gain, eps, up):
    d = x.shape[-1]
    mean = x.mean(-1, keepdims=True)
    c = x - mean
    var = (c * c).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = c * rstd
    dxhat = up * gain
    s1 = dxhat.sum(-1, keepdims=True)
    s2 = (dxhat * xhat).sum(-1, keepdims=True)
    dx = rstd * (dxhat - s1 / d - xhat * (s2 / d))
    dgain = (up * xhat).reshape(-1, d).sum(0)
    dbias = up.reshape(-1, d).sum(0)
    return dx, dgain, dbias


def gelu(v):
    t = np.tanh(GELU_C * (v + GELU_A * v * v * v))
    return 0.5 * v * (1.0 + t)


def gelu_vjp(v, up):
    t = np.tanh(GELU_C * (v + GELU_A * v * v * v))
    dt = (1.0 - t * t) * GELU_C * (1.0 + 3.0 * GELU_A * v * v)
    return up * (0.5 * (1.0 + t) + 0.5 * v * dt)


def softmax_rows(s):
    m = s.max(-1, keepdims=True)
    e = np.exp(s - m)
    return e / e.sum(-1, keepdims=True)


# ---------------------------------------------------------------------------
# attention (blocks.cpp:142-236), batched over samples
# ---------------------------------------------------------------------------


def _heads(t, H):
    B, s, d = t.shape
    return t.reshape(B, s, H, d // H).transpose(0, 2, 1, 3)


def _merge(t):
    B, H, s, dh = t.shape
    return t.transpose(0, 2, 1, 3).reshape(B, s, H * dh)


def _attn_probs(q, k, causal, inv_s):
    sc = (q @ k.transpose(0, 1, 3, 2)) * inv_s
    if causal:
        sq, sk = sc.shape[-2:]
        sc = sc + np.triu(np.full((sq, sk), KMASK), 1)
    return softmax_rows(sc)


def attention(p, prefix, H, causal, xq, xkv):
    d = xq.shape[-1]
    inv_s = 1.0 / math.sqrt(d // H)
    q = _heads(linear(xq, p[prefix + ".q.w"], p[prefix + ".q.b"]), H)
    k = _heads(linear(xkv, p[prefix + ".k.w"], p[prefix + ".k.b"]), H)
    v = _heads(linear(xkv, p[prefix + ".v.w"], p[prefix + ".v.b"]), H)
    P = _attn_probs(q, k, causal, inv_s)
    ctx = _merge(P @ v)
    return linear(ctx, p[prefix + ".o.w"], p[prefix + ".o.b"])


def _acc(g, name, gscale, val):
    if g is not None:
        g[name] += gscale * val


def _linear_vjp(x, w, up, g, name, gscale):
    dx = up @ w
    if g is not None:
        d_out = w.shape[0]
        g[name + ".w"] += gscale * (up.reshape(-1, d_out).T @ x.reshape(-1, x.shape[-1]))
        g[name + ".b"] += gscale * up.reshape(-1, d_out).sum(0)
    return dx


def attention_vjp(p, prefix, H, causal, xq, xkv, up, g, gscale):
    d = xq.shape[-1]
    inv_s = 1.0 / math.sqrt(d // H)
    q = _heads(linear(xq, p[prefix + ".q.w"], p[prefix + ".q.b"]), H)
    k = _heads(linear(xkv, p[prefix + ".k.w"], p[prefix + ".k.b"]), H)
    v = _heads(linear(xkv, p[prefix + ".v.w"], p[prefix + ".v.b"]), H)
    P = _attn_probs(q, k, causal, inv_s)
    ctx = _merge(P @ v)
    dctx = _linear_vjp(ctx, p[prefix + ".o.w"], up, g, prefix + ".o", gscale)
    dctx_h = _heads(dctx, H)
    dP = dctx_h @ v.transpose(0, 1, 3, 2)
    dv = P.transpose(0, 1, 3, 2) @ dctx_h
    t = (dP * P).sum(-1, keepdims=True)
    dS = P * (dP - t)
    dq = (dS @ k) * inv_s
    dk = (dS.transpose(0, 1, 3, 2) @ q) * inv_s
    dxq = _linear_vjp(xq, p[prefix + ".q.w"], _merge(dq), g, prefix + ".q", gscale)
    dxk = _linear_vjp(xkv, p[prefix + ".k.w"], _merge(dk), g, prefix + ".k", gscale)
    dxv = _linear_vjp(xkv, p[prefix + ".v.w"], _merge(dv), g, prefix + ".v", gscale)
    return dxq, dxk + dxv


def _ln_vjp(x, p, name, eps, up, g, gscale):
    dx, dg, db = layer_norm_vjp(x, p[name + ".gain"], eps, up)
    _acc(g, name + ".gain", gscale, dg)
    _acc(g, name + ".bias", gscale, db)
    return dx


def _mlp(p, x):
    return linear(gelu(linear(x, p["mlp.in.w"], p["mlp.in.b"])), p["mlp.out.w"], p["mlp.out.b"])


def _mlp_vjp(p, x, up, g, gscale):
    a = linear(x, p["mlp.in.w"], p["mlp.in.b"])
    ga = gelu(a)
    dga = _linear_vjp(ga, p["mlp.out.w"], up, g, "mlp.out", gscale)
    da = gelu_vjp(a, dga)
    return _linear_vjp(x, p["mlp.in.w"], da, g, "mlp.in", gscale)


# ---------------------------------------------------------------------------
# block residuals (blocks.cpp:246-333)
# ---------------------------------------------------------------------------


def encoder_residual(p, H, causal, eps, x):
    n1 = layer_norm(x, p["ln1.gain"], p["ln1.bias"], eps)
    a1 = attention(p, "attn", H, causal, n1, n1)
    u = x + a1
    n2 = layer_norm(u, p["ln2.gain"], p["ln2.bias"], eps)
    return a1 + _mlp(p, n2)


def encoder_residual_vjp(p, H, causal, eps, x, up, g, gscale):
    n1 = layer_norm(x, p["ln1.gain"], p["ln1.bias"], eps)
    a1 = attention(p, "attn", H, causal, n1, n1)
    u = x + a1
    n2 = layer_norm(u, p["ln2.gain"], p["ln2.bias"], eps)
    dn2 = _mlp_vjp(p, n2, up, g, gscale)
    du = _ln_vjp(u, p, "ln2", eps, dn2, g, gscale)
    dx = du
    da1 = up + du
    dq, dkv = attention_vjp(p, "attn", H, causal, n1, n1, da1, g, gscale)
    return dx + _ln_vjp(x, p, "ln1", eps, dq + dkv, g, gscale)


def decoder_residual(p, H, eps, y, xe):
    n1 = layer_norm(y, p["ln1.gain"], p["ln1.bias"], eps)
    a1 = attention(p, "self", H, True, n1, n1)
    u3 = y + a1
    n3 = layer_norm(u3, p["ln3.gain"], p["ln3.bias"], eps)
    c = attention(p, "cross", H, False, n3, xe)
    ybar = a1 + c
    u2 = y + ybar
    n2 = layer_norm(u2, p["ln2.gain"], p["ln2.bias"], eps)
    return ybar + _mlp(p, n2)


def decoder_residual_vjp(p, H, eps, y, xe, up, g, gscale):
    n1 = layer_norm(y, p["ln1.gain"], p["ln1.bias"], eps)
    a1 = attention(p, "self", H, True, n1, n1)
    u3 = y + a1
    n3 = layer_norm(u3, p["ln3.gain"], p["ln3.bias"], eps)
    c = attention(p, "cross", H, False, n3, xe)
    ybar = a1 + c
    u2 = y + ybar
    n2 = layer_norm(u2, p["ln2.gain"], p["ln2.bias"], eps)
    dn2 = _mlp_vjp(p, n2, up, g, gscale)
    du2 = _ln_vjp(u2, p, "ln2", eps, dn2, g, gscale)
    dy = du2
    dybar = up + du2
    da1 = dybar
    cq, ckv = attention_vjp(p, "cross", H, False, n3, xe, dybar, g, gscale)
    du3 = _ln_vjp(u3, p, "ln3", eps, cq, g, gscale)
    dy = dy + du3
    da1 = da1 + du3
    sq, skv = attention_vjp(p, "self", H, True, n1, n1, da1, g, gscale)
    dy = dy + _ln_vjp(y, p, "ln1", eps, sq + skv, g, gscale)
    return dy, ckv


# ---------------------------------------------------------------------------
# serial sweeps (blocks.cpp:659-682)
# ---------------------------------------------------------------------------


def serial_forward(stack: Stack, z0: State) -> List[State]:
    traj = [z0]
    for n in range(stack.total):
        traj.append(stack.step(n, stack.h[n], traj[-1]))
    return traj


def serial_adjoint(stack: Stack, traj, lam_n: State, grads=None) -> List[State]:
    lam = [None] * (stack.total + 1)
    lam[stack.total] = lam_n
    for n in range(stack.total - 1, -1, -1):
        h = stack.h[n]
        lam[n] = stack.adjoint_step(n, h, traj[n], lam[n + 1], grads, h)
    return lam


# ---------------------------------------------------------------------------
# MGRIT (mgrit.hpp:58-303)
# ---------------------------------------------------------------------------


class ScalarLinearSystem:
    """systems.hpp:30-71."""

    def __init__(self, rates, h, cf):
        self.rates = list(rates)
        self.h = h
        self.cf = cf

    def phi(self, level, k, z):
        stride = self.cf ** level
        dt = float(stride) * self.h
        return z + dt * self.rates[k * stride] * z

    add = staticmethod(lambda a, b: a + b)
    sub = staticmethod(lambda a, b: a - b)
    zeros_like = staticmethod(lambda s: 0.0)
    norm_sq = staticmethod(lambda s: s * s)


class StackForwardSystem:
    """systems.hpp:80-102."""

    def __init__(self, stack: Stack, cf):
        self.stack, self.cf = stack, cf

    def phi(self, level, k, z):
        stride = self.cf ** level
        layer = self.stack.ib + k * stride
        return self.stack.step(layer, stride * self.stack.interior_h(), z)

    add = staticmethod(lambda a, b: a + b)
    sub = staticmethod(lambda a, b: a - b)
    zeros_like = staticmethod(lambda s: s.zeros_like())
    norm_sq = staticmethod(lambda s: s.norm_sq())


class StackAdjointSystem:
    """adjoint.hpp:35-65: step m applies layer N-1-m^T at traj[N-1-m]."""

    def __init__(self, stack: Stack, cf):
        self.stack, self.cf = stack, cf
        self.traj = []

    def phi(self, level, k, mu):
        stride = self.cf ** level
        n = len(self.traj) - 1 - 1 - k * stride
        if n < 0 or n >= len(self.traj) - 1:
            raise RuntimeError("StackAdjointSystem: step outside the recorded trajectory")
        layer = self.stack.ib + n
        return self.stack.adjoint_step(layer, stride * self.stack.interior_h(), self.traj[n], mu,
                                       None, 0.0)

    add = staticmethod(lambda a, b: a + b)
    sub = staticmethod(lambda a, b: a - b)
    zeros_like = staticmethod(lambda s: s.zeros_like())
    norm_sq = staticmethod(lambda s: s.norm_sq())


class ValidationError(ValueError):
    pass


class _Level:
    def __init__(self, n, coarse):
        self.n = n
        self.v = [None] * (n + 1)
        if coarse:
            self.base = [None] * (n + 1)
            self.rho = [None] * (n + 1)
            self.phib = [None] * (n + 1)


class MgritSolver:
    """mgrit.hpp:58-303 (FCF relaxation, FAS coarse levels, exact coarsest solve)."""

    def __init__(self, sys, n_steps, cf, levels):
        if cf < 2:
            raise ValidationError("MgritSolver: coarsening factor must be >= 2")
        if levels < 1:
            raise ValidationError("MgritSolver: need at least one level")
        if n_steps < 1:
            raise ValidationError("MgritSolver: need at least one step")
        stride = 1
        for _ in range(max(levels - 1, 1)):
            stride *= cf
            if stride > n_steps:
                raise ValidationError("MgritSolver: too many levels")
        if n_steps % stride:
            raise ValidationError("MgritSolver: step count must be divisible by coarsen^(levels-1)")
        self.sys, self.cf, self.L = sys, cf, levels
        self.lv = []
        n = n_steps
        for l in range(levels):
            self.lv.append(_Level(n, l > 0))
            if l + 1 < levels:
                n //= cf
        self.phi_calls = 0

    def states(self, level=0):
        return self.lv[level].v

    def set_initial_condition(self, z0):
        self.lv[0].v[0] = z0

    def apply_initial_guess(self, policy):
        f = self.lv[0]
        if policy == "broadcast":
            for j in range(1, f.n + 1):
                f.v[j] = f.v[0]
        elif policy == "zero":
            for j in range(1, f.n + 1):
                f.v[j] = self.sys.zeros_like(f.v[0])

    def _phi(self, level, k, z):
        self.phi_calls += 1
        return self.sys.phi(level, k, z)

    def relax_update(self, level, j):
        lev = self.lv[level]
        p = self._phi(level, j - 1, lev.v[j - 1])
        if level == 0:
            lev.v[j] = p
        else:
            corr = self.sys.add(self.sys.sub(p, lev.phib[j]), lev.rho[j])
            lev.v[j] = self.sys.add(lev.base[j], corr)

    def f_relax(self, level):
        lev = self.lv[level]
        for k in range(lev.n // self.cf):
            for i in range(1, self.cf):
                self.relax_update(level, k * self.cf + i)

    def c_relax(self, level):
        lev = self.lv[level]
        for k in range(1, lev.n // self.cf + 1):
            self.relax_update(level, k * self.cf)

    def fcf_relax(self, level):
        self.f_relax(level)
        self.c_relax(level)
        self.f_relax(level)

    def residual_rows(self, level):
        lev, s = self.lv[level], self.sys
        r = [None] * (lev.n + 1)
        if level == 0:
            r[0] = s.zeros_like(lev.v[0])
        else:
            r[0] = s.add(s.sub(lev.base[0], lev.v[0]), lev.rho[0])
        for j in range(1, lev.n + 1):
            p = self._phi(level, j - 1, lev.v[j - 1])
            if level == 0:
                r[j] = s.sub(p, lev.v[j])
            else:
                lhs = s.add(s.sub(p, lev.phib[j]), lev.rho[j])
                r[j] = s.sub(lhs, s.sub(lev.v[j], lev.base[j]))
        return r

    def norm_of(self, rows):
        # plain left-to-right accumulation (mgrit.hpp:189-193); Python's
        # built-in sum() is compensated since 3.12 and would differ
        s = 0.0
        for x in rows:
            s += self.sys.norm_sq(x)
        return math.sqrt(s)

    def restrict_to(self, level, fine_rows):
        c, f = self.lv[level], self.lv[level - 1]
        for k in range(c.n + 1):
            c.base[k] = f.v[k * self.cf]
            c.rho[k] = fine_rows[k * self.cf]
            c.v[k] = c.base[k]
        for k in range(1, c.n + 1):
            c.phib[k] = self._phi(level, k - 1, c.base[k - 1])

    def correct_from(self, level):
        c, f = self.lv[level], self.lv[level - 1]
        for k in range(1, c.n + 1):
            e = self.sys.sub(c.v[k], c.base[k])
            f.v[k * self.cf] = self.sys.add(f.v[k * self.cf], e)

    def exact_solve(self, level):
        lev = self.lv[level]
        lev.v[0] = lev.base[0]
        for j in range(1, lev.n + 1):
            self.relax_update(level, j)

    def _descend(self, level):
        if level == self.L - 1:
            self.exact_solve(level)
            return
        self.fcf_relax(level)
        rows = self.residual_rows(level)
        self.restrict_to(level + 1, rows)
        self._descend(level + 1)
        self.correct_from(level + 1)
        self.f_relax(level)

    def v_cycle(self):
        self.fcf_relax(0)
        rows = self.residual_rows(0)
        nrm = self.norm_of(rows)
        if self.L > 1:
            self.restrict_to(1, rows)
            self._descend(1)
            self.correct_from(1)
            self.f_relax(0)
        return nrm

    def solve_forward(self, max_iters, tol):
        if max_iters < 1:
            raise ValidationError("solve_forward: need at least one iteration")
        trace, conv = [], False
        for _ in range(max_iters):
            nrm = self.v_cycle()
            trace.append(nrm)
            if not math.isfinite(nrm):
                break
            if nrm <= tol * trace[0]:
                conv = True
                break
        return trace, conv


# ---------------------------------------------------------------------------
# engine (adjoint.hpp:70-219)
# ---------------------------------------------------------------------------


@dataclass
class SolveConfig:
    coarsen: int = 2
    levels: int = 2
    fwd_iters: int = 2
    bwd_iters: int = 1
    fwd_tol: float = 0.0
    bwd_tol: float = 0.0
    cold_guess: str = "broadcast"
    warm_start: bool = True


class LayerParallelEngine:
    def __init__(self, stack: Stack, cfg: SolveConfig):
        self.stack, self.cfg = stack, cfg
        n = stack.interior_layers
        self.fwd_sys = StackForwardSystem(stack, cfg.coarsen)
        self.adj_sys = StackAdjointSystem(stack, cfg.coarsen)
        self.fwd = MgritSolver(self.fwd_sys, n, cfg.coarsen, cfg.levels)
        self.bwd = MgritSolver(self.adj_sys, n, cfg.coarsen, cfg.levels)
        self.first_fwd = self.first_bwd = True

    def forward(self, z0: State):
        st, cfg = self.stack, self.cfg
        traj = [None] * (st.total + 1)
        traj[0] = z0
        for l in range(st.ib):
            traj[l + 1] = st.step(l, st.h[l], traj[l])
        self.fwd.set_initial_condition(traj[st.ib])
        self.fwd.apply_initial_guess(cfg.cold_guess if (self.first_fwd or not cfg.warm_start)
                                     else "warm")
        self.first_fwd = False
        trace, conv = self.fwd.solve_forward(cfg.fwd_iters, cfg.fwd_tol)
        n = st.interior_layers
        for j in range(n + 1):
            traj[st.ib + j] = self.fwd.states(0)[j]
        for l in range(st.ie, st.total):
            traj[l + 1] = st.step(l, st.h[l], traj[l])
        return traj, trace, conv

    def backward(self, traj, lam_n: State, grads=None):
        st, cfg = self.stack, self.cfg
        lam = lam_n
        for l in range(st.total - 1, st.ie - 1, -1):
            lam = st.adjoint_step(l, st.h[l], traj[l], lam, grads, st.h[l])
        n = st.interior_layers
        self.adj_sys.traj = traj[st.ib:st.ib + n + 1]
        self.bwd.set_initial_condition(lam)
        self.bwd.apply_initial_guess(cfg.cold_guess if (self.first_bwd or not cfg.warm_start)
                                     else "warm")
        self.first_bwd = False
        trace, conv = self.bwd.solve_forward(cfg.bwd_iters, cfg.bwd_tol)
        mu = self.bwd.states(0)
        if grads is not None:
            h = st.interior_h()
            for i in range(n):
                layer = st.ib + i
                st.residual_vjp(layer, traj[layer], mu[n - 1 - i], grads, h)
        lam = mu[n]
        for l in range(st.ib - 1, -1, -1):
            lam = st.adjoint_step(l, st.h[l], traj[l], lam, grads, st.h[l])
        return lam, trace, conv


# ---------------------------------------------------------------------------
# controller (controller.hpp:63-155)
# ---------------------------------------------------------------------------

KEEP, INCREASE, SWITCH = 0, 1, 2


def last_pair_factor(trace):
    n = len(trace)
    if n < 2 or trace[n - 2] == 0.0:
        return 0.0
    return trace[n - 1] / trace[n - 2]


def decide(f_fwd, f_bwd, threshold, policy_switch, cap, fwd_iters, bwd_iters):
    if threshold <= 0.0:
        raise ValidationError("decide: threshold must be positive")
    worst = max(f_fwd, f_bwd)
    if worst <= threshold:
        return KEEP
    if policy_switch:
        return SWITCH
    return INCREASE if (fwd_iters < cap or bwd_iters < cap) else SWITCH
