"""Generates the full-depth parity fixtures tests/golden/deep_<config>.npz (and
bench_bert_traces.npz) in the build container. Run:

    python tests/golden/make_deep.py [name ...]

The outputs come from the float64 numpy restatement oracle/mglp_oracle.py
(LayerParallelEngine.forward / backward, adjoint.hpp:113-183), which
tests/test_oracle.py pins to <1e-12 of the compiled reference
(oracle/_ref/libmglp_ref.so); the parameters are the compiled reference's
own LayerStack(cfg, seed=7) initialisation (blocks.cpp:432-449), and z0 /
lambda_N come from the compiled rng::gaussian (rng.hpp:70-94). The compiled
reference's scalar matmul is too slow at these sizes (0.9 s per
step at B=1), the numpy port runs the same algorithm with BLAS.
Summaries: tests/_deep.py.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))
from oracle import mglp_oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402
import _deep as D  # noqa: E402


def oracle_stack(c, seed=7):
    rc = R.RefStackConfig(kind=c["kind"], d=c["d"], heads=c["heads"], ffn=c["ffn"],
                          n_enc=c["n_enc"], n_dec=c["n_dec"])
    rs = R.RefStack(rc, seed)
    flat = rs.get_params()
    del rs
    st = O.Stack(O.StackConfig(kind=c["kind"], d=c["d"], heads=c["heads"], ffn=c["ffn"],
                               n_enc=c["n_enc"], n_dec=c["n_dec"]), flat)
    return st, flat


def inputs(c):
    n = D.state_len(c)
    z0 = R.gaussian_fill(7, D.K_TEST, 7, n, 0.5)
    lam = R.gaussian_fill(8, D.K_TEST, 8, n, 1.0)
    return z0, lam


def run(c, grads=True):
    st, flat = oracle_stack(c)
    z0, lam = inputs(c)
    sf = lambda a: O.State.from_flat(a, c["B"], c["sx"], c["sy"], c["d"])  # noqa: E731
    eng = O.LayerParallelEngine(st, O.SolveConfig(coarsen=c["cf"], levels=c["levels"],
                                                  fwd_iters=c["fwd_iters"],
                                                  bwd_iters=c["bwd_iters"], warm_start=False))
    t0 = time.time()
    traj, ftr, _ = eng.forward(sf(z0))
    t1 = time.time()
    g = st.zero_grads() if grads else None
    lam0, btr, _ = eng.backward(traj, sf(lam), g)
    t2 = time.time()
    print(f"  forward {t1 - t0:.0f}s backward {t2 - t1:.0f}s  fwd {ftr} bwd {btr}", flush=True)
    return st, traj, ftr, btr, lam0, g


def make(name, c):
    print(name, flush=True)
    st, traj, ftr, btr, lam0, g = run(c)
    flat_traj = [t.flat() for t in traj]
    out = dict(meta=json.dumps(dict(c, name=name, seed=7)), fwd_trace=np.array(ftr),
               bwd_trace=np.array(btr), lam0=lam0.flat().astype(np.float32),
               lam0_norm=np.array([np.linalg.norm(lam0.flat())]),
               traj_last=flat_traj[-1].astype(np.float32))
    out.update(D.state_summary(c, flat_traj))
    out.update(D.grad_summary(c, O.Stack.flatten(g)))
    path = os.path.join(HERE, f"deep_{name.replace('_deep', '')}.npz")
    np.savez_compressed(path, **out)
    print(f"  -> {path} {os.path.getsize(path) / 1024:.0f} KiB", flush=True)


def make_bench_traces():
    c = D.BENCH_BERT
    print("bench_bert (B=32)", flush=True)
    st, traj, ftr, btr, lam0, _ = run(c, grads=False)
    flat_traj = [t.flat() for t in traj]
    s = D.state_summary(c, [flat_traj[-1]])
    lam0f = lam0.flat()
    idx = s["s_idx"]
    out = dict(meta=json.dumps(dict(c, name="bench_bert", seed=7)), fwd_trace=np.array(ftr),
               bwd_trace=np.array(btr), traj_last_norm=s["s_norm"], traj_last_samp=s["s_samp"][0],
               lam0_norm=np.array([np.linalg.norm(lam0f)]), lam0_samp=lam0f[idx], s_idx=idx)
    path = os.path.join(HERE, "bench_bert_traces.npz")
    np.savez_compressed(path, **out)
    print(f"  -> {path} {os.path.getsize(path) / 1024:.0f} KiB", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or list(D.DEEP) + ["bench_bert"]
    for nm in names:
        if nm == "bench_bert":
            make_bench_traces()
        else:
            make(nm, D.DEEP[nm])
