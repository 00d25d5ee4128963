"""Full-depth parity at every BASELINE config's own depth, width, heads,
sequence length, c_f and hierarchy, through the C-ABI,
against tests/golden/deep_*.npz and bench_bert_traces.npz (made by
tests/golden/make_deep.py from the float64 numpy oracle, itself pinned
<1e-12 to the compiled reference in tests/test_oracle.py):

  BERT 64L  d=768 s=128  c_f=4 2 levels      (configs[1])
  GPT  128L d=768 s=512  causal, c_f=4 3 lvl (configs[2])
  ViT  64L  d=768 s=197  c_f=8 2 levels      (configs[3])
  MT   32+32 d=512 s=128 one stacked solve   (configs[4])

at batch 1, one forward + one adjoint V-cycle + the parameter pass (the
bench's hierarchy), plus the bench's own BERT workload at batch 32 (both
first-cycle traces, lambda_0, the final state).

Checked, each at the north-star tolerance 1e-4 (relative):
  * both residual traces;
  * lambda_0 and the final state, every entry (max |dev - ref| / max |ref|);
  * every trajectory state: its L2 norm and 2048 fixed entries;
  * every (layer, parameter tensor) gradient: its L2 norm, 128 fixed entries
    (relative to the tensor's max |g|) and the Frobenius norm of the WHOLE
    error estimated by 8 Rademacher sketches (tests/_deep.py).
Tensors whose exact gradient vanishes (the attention key bias: softmax is
shift invariant; the f64 reference holds ~1e-15 against O(10) gradients
elsewhere in the layer) hold rounding noise on both sides; they are measured
against their layer's largest gradient, every other tensor against its own
(floored at 1e-3 of the layer's largest).
Set MGLP_PARITY_REPORT=<path> to write the per-config errors as JSON.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

import _deep as D
from paper_2601_09026_b200 import _native as N
from paper_2601_09026_b200.engine import SolveConfig, StackConfig

pytestmark = pytest.mark.gpu
TOL = 1e-4
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_REPORT = {}


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(float(np.abs(b).max()), 1e-300))


def run_device(c, want_grads=True):
    import torch
    sc = StackConfig(kind=c["kind"], d=c["d"], heads=c["heads"], ffn=c["ffn"], n_enc=c["n_enc"],
                     n_dec=c["n_dec"])
    so = SolveConfig(coarsen=c["cf"], levels=c["levels"], fwd_iters=c["fwd_iters"],
                     bwd_iters=c["bwd_iters"], warm_start=False)
    h = C.c_void_p()
    N.call("mglp_engine_create", C.byref(sc.desc()), C.byref(so.desc()), 0, C.byref(h))
    try:
        N.call("mglp_engine_init_params", h, C.c_ulonglong(7), None)
        ns = C.c_longlong()
        N.call("mglp_engine_set_shape", h, c["B"], c["sx"], c["sy"], C.byref(ns))
        n = D.state_len(c)
        z0h, lamh = np.empty(n), np.empty(n)
        N.call("mglp_rng_gaussian_fill", 7, D.K_TEST, 7, 0.5, N.dptr(z0h), n)
        N.call("mglp_rng_gaussian_fill", 8, D.K_TEST, 8, 1.0, N.dptr(lamh), n)
        dev = torch.device("cuda", 0)
        z0 = torch.zeros(ns.value, dtype=torch.float32, device=dev)
        lam = torch.zeros_like(z0)
        lam0 = torch.zeros_like(z0)
        z0[:n] = torch.from_numpy(z0h).float()
        lam[:n] = torch.from_numpy(lamh).float()
        torch.cuda.synchronize()
        N.call("mglp_engine_zero_grads", h)
        N.call("mglp_engine_forward_device", h, C.c_void_p(z0.data_ptr()))
        N.call("mglp_engine_backward_device", h, C.c_void_p(lam.data_ptr()),
               C.c_void_p(lam0.data_ptr()), 1 if want_grads else 0)
        tr = np.empty(64)
        nt, cv = C.c_int(), C.c_int()
        N.call("mglp_engine_trace", h, 0, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
        ftr = tr[:nt.value].copy()
        N.call("mglp_engine_trace", h, 1, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
        btr = tr[:nt.value].copy()
        total = c["n_enc"] + c["n_dec"]
        traj = torch.empty((total + 1) * ns.value, dtype=torch.float32, device=dev)
        N.call("mglp_engine_read_traj", h, 0, total + 1, C.c_void_p(traj.data_ptr()))
        traj_h = traj.view(total + 1, ns.value)[:, :n].double().cpu().numpy()
        out = dict(fwd_trace=ftr, bwd_trace=btr, lam0=lam0[:n].double().cpu().numpy(),
                   traj=traj_h)
        if want_grads:
            flat = []
            for layer in range(total):
                cnt = sum(sz for _, sz in D.components(c["kind"], c["n_enc"], c["d"], c["ffn"],
                                                         layer))
                g = np.zeros(cnt)
                N.call("mglp_engine_get_grads_layers", h, layer, layer + 1, N.dptr(g), cnt)
                flat.append(g)
            out["grads"] = np.concatenate(flat)
        return out
    finally:
        N.call("mglp_engine_destroy", h)


def grad_errors(c, dev_flat, ref):
    d = D.grad_summary(c, dev_flat)
    total = c["n_enc"] + c["n_dec"]
    ncomp = [len(D.components(c["kind"], c["n_enc"], c["d"], c["ffn"], l)) for l in range(total)]
    def per_layer_max(v):
        out, o = [], 0
        for k in ncomp:
            out.append(np.full(k, v[o:o + k].max()))
            o += k
        return np.concatenate(out)

    # tensors whose exact gradient vanishes identically (the attention key
    # bias, softmax shift invariance: the f64 reference holds ~1e-15 noise of
    # a layer whose gradients are O(10-100)) carry only rounding noise on both
    # sides; they are measured against their layer's scale, all others against
    # their own (floored at 1e-3 of the layer's largest)
    def floor_of(v):
        lm = per_layer_max(v)
        return np.where(v < 1e-9 * lm, lm, np.maximum(v, 1e-3 * lm))

    den = floor_of(ref["g_norm"])
    sketch = np.sqrt(np.mean((d["g_sketch"] - ref["g_sketch"]) ** 2, axis=1)) / den
    norm = np.abs(d["g_norm"] - ref["g_norm"]) / den
    # sampled entries relative to each tensor's max |g| (same floor)
    sizes = [min(sz, D.N_GRAD_IDX) for l in range(total)
             for _, sz in D.components(c["kind"], c["n_enc"], c["d"], c["ffn"], l)]
    gden = floor_of(ref["g_max"])
    samp = np.abs(d["g_samp"] - ref["g_samp"]) / np.repeat(gden, sizes)
    names = [f"layer {l} {nm}" for l in range(total)
             for nm, _ in D.components(c["kind"], c["n_enc"], c["d"], c["ffn"], l)]
    owner = np.repeat(np.arange(len(names)), sizes)
    ws = int(owner[int(np.argmax(samp))])
    return dict(grad_sketch_frobenius=float(sketch.max()), grad_norms=float(norm.max()),
                grad_samples=float(samp.max()), grad_tensors=int(sketch.size),
                worst_sketch=names[int(np.argmax(sketch))], worst_norm=names[int(np.argmax(norm))],
                worst_sample=f"{names[ws]} (|g|max {ref['g_max'][ws]:.3e}, floor "
                             f"{gden[ws]:.3e}, norm {ref['g_norm'][ws]:.3e})")


def _report(name, errs):
    _REPORT[name] = errs
    path = os.environ.get("MGLP_PARITY_REPORT")
    if path:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump(dict(tolerance=TOL, configs=_REPORT), f, indent=1, sort_keys=True)


@pytest.mark.parametrize("name", ["bert_deep", "gpt_deep", "vit_deep", "mt_deep"])
def test_full_depth_against_oracle(name):
    path = os.path.join(GOLDEN, f"deep_{name.replace('_deep', '')}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    ref = np.load(path)
    c = json.loads(str(ref["meta"]))
    out = run_device(c)
    s = D.state_summary(c, out["traj"])
    smax = np.abs(ref["s_samp"]).max(axis=1, keepdims=True)
    errs = dict(
        fwd_trace=rel(out["fwd_trace"], ref["fwd_trace"]),
        bwd_trace=rel(out["bwd_trace"], ref["bwd_trace"]),
        lambda0=rel(out["lam0"], ref["lam0"]),
        traj_last=rel(out["traj"][-1], ref["traj_last"]),
        state_norms=float((np.abs(s["s_norm"] - ref["s_norm"]) / ref["s_norm"]).max()),
        state_samples=float((np.abs(s["s_samp"] - ref["s_samp"]) / smax).max()),
        n_states=int(ref["s_norm"].size),
    )
    errs.update(grad_errors(c, out["grads"], ref))
    errs["config"] = {k: c[k] for k in ("kind", "n_enc", "n_dec", "d", "heads", "sx", "sy", "B",
                                        "cf", "levels", "fwd_iters", "bwd_iters")}
    _report(name, errs)
    bad = {k: v for k, v in errs.items() if isinstance(v, float) and not v <= TOL}
    assert not bad, (name, errs)


def test_bench_bert_traces_against_oracle():
    """The bench's own workload (configs[1], batch 32): first-cycle forward
    and adjoint residual norms, lambda_0 and the final state."""
    path = os.path.join(GOLDEN, "bench_bert_traces.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    ref = np.load(path)
    c = json.loads(str(ref["meta"]))
    out = run_device(c, want_grads=False)
    idx = ref["s_idx"]
    errs = dict(
        fwd_trace=rel(out["fwd_trace"], ref["fwd_trace"]),
        bwd_trace=rel(out["bwd_trace"], ref["bwd_trace"]),
        lambda0_norm=abs(np.linalg.norm(out["lam0"]) - ref["lam0_norm"][0]) / ref["lam0_norm"][0],
        lambda0_samples=rel(out["lam0"][idx], ref["lam0_samp"]),
        traj_last_norm=abs(np.linalg.norm(out["traj"][-1]) - ref["traj_last_norm"][0])
        / ref["traj_last_norm"][0],
        traj_last_samples=rel(out["traj"][-1][idx], ref["traj_last_samp"]),
        device_fwd_trace=[float(x) for x in out["fwd_trace"]],
        oracle_fwd_trace=[float(x) for x in ref["fwd_trace"]],
        device_bwd_trace=[float(x) for x in out["bwd_trace"]],
        oracle_bwd_trace=[float(x) for x in ref["bwd_trace"]],
    )
    _report("bench_bert_B32", errs)
    bad = {k: v for k, v in errs.items() if isinstance(v, float) and not v <= TOL}
    assert not bad, errs
