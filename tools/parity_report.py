"""Measured device-vs-reference errors (max|d-r|/max|r|) for every golden
fixture and a full-width BERT slice; writes gpurun_out/parity_report.json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import mglp_oracle as O  # noqa: E402
from paper_2601_09026_b200 import (LayerParallelEngine, LayerStack, SolveConfig,  # noqa: E402
                                   StackConfig, State, serial_adjoint, serial_forward)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


out = {}
for name in ["enc_small", "enc_small_3lvl", "causal_buffered", "encdec", "tiny_baseline"]:
    g = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
    m = json.loads(str(g["meta"]))
    sc = StackConfig(kind=m["kind"], d=m["d"], heads=m["heads"], ffn=m["ffn"], n_enc=m["n_enc"],
                     n_dec=m["n_dec"], buffer_open=m["buffer_open"], buffer_close=m["buffer_close"])
    st = LayerStack(sc, m["seed"])
    if "params" in g:
        st.set_params(g["params"])
    sf = lambda a: State.from_flat(a, m["B"], m["sx"], m["sy"], m["d"])  # noqa: E731
    eng = LayerParallelEngine(st, SolveConfig(coarsen=m["cf"], levels=m["levels"],
                                              fwd_iters=m["fwd_iters"], bwd_iters=m["bwd_iters"],
                                              warm_start=False))
    fo = eng.forward(sf(g["z0"]))
    gr = st.zero_grads()
    bo = eng.backward(fo.traj, sf(g["lamN"]), gr)
    r = {"fwd_trace": rel(fo.phase.trace, g["fwd_trace"]),
         "bwd_trace": rel(bo.phase.trace, g["bwd_trace"]),
         "lambda0": rel(bo.lambda0.flat(), g["lam0"])}
    if "traj" in g:
        r["traj"] = rel(np.stack([t.flat() for t in fo.traj]), g["traj"])
        r["grads"] = rel(gr, g["grads"])
        traj = serial_forward(st, sf(g["z0"]))
        r["serial_traj"] = rel(np.stack([t.flat() for t in traj]), g["serial_traj"])
        sg = st.zero_grads()
        lam = serial_adjoint(st, traj, sf(g["lamN"]), sg)
        r["serial_grads"] = rel(sg, g["serial_grads"])
    else:
        r["traj_last"] = rel(fo.traj[-1].flat(), g["traj_last"])
        r["grads_head"] = rel(gr[:4096], g["grads_head"])
    out[name] = r
    print(name, json.dumps(r), flush=True)

# full width (d=768, 12 heads, ffn 3072) vs the numpy oracle: seq 128 on 8
# layers (fused short attention, pre-split P), and the streamed long attention
# at GPT-2 (causal, 512) and ViT (197) lengths on 4 layers
for kind, s, B, nl in [("encoder", 128, 2, 8), ("decoder_only", 128, 2, 8),
                       ("decoder_only", 512, 1, 4), ("encoder", 197, 1, 4)]:
    kw = dict(n_enc=nl) if kind == "encoder" else dict(n_dec=nl)
    sc = StackConfig(kind=kind, d=768, heads=12, ffn=3072, **kw)
    st = LayerStack(sc, 7)
    ost = O.Stack(O.StackConfig(kind=kind, d=768, heads=12, ffn=3072, **kw), np.asarray(st.params()))
    rng = np.random.default_rng(3)
    z0 = rng.standard_normal(B * s * 768) * 0.5
    lam = rng.standard_normal(B * s * 768)
    cfg = dict(coarsen=4 if nl == 8 else 2, levels=2, fwd_iters=2, bwd_iters=1)
    eng = LayerParallelEngine(st, SolveConfig(**cfg))
    fo = eng.forward(State.from_flat(z0, B, s, 0, 768))
    gr = st.zero_grads()
    bo = eng.backward(fo.traj, State.from_flat(lam, B, s, 0, 768), gr)
    oe = O.LayerParallelEngine(ost, O.SolveConfig(**cfg))
    otraj, otr, _ = oe.forward(O.State.from_flat(z0, B, s, 0, 768))
    og = ost.zero_grads()
    ol0, obtr, _ = oe.backward(otraj, O.State.from_flat(lam, B, s, 0, 768), og)
    r = {"traj": rel(np.stack([t.flat() for t in fo.traj]), np.stack([t.flat() for t in otraj])),
         "fwd_trace": rel(fo.phase.trace, otr), "bwd_trace": rel(bo.phase.trace, obtr),
         "lambda0": rel(bo.lambda0.flat(), ol0.flat()), "grads": rel(gr, O.Stack.flatten(og))}
    key = f"full_width_{kind}_{nl}L" if s == 128 else f"full_width_{kind}_s{s}_{nl}L"
    out[key] = r
    print(key, json.dumps(r), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "parity_report.json"), "w"), indent=1)
