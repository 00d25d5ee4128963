"""Generates the golden fixtures under tests/golden/ by running the COMPILED
REFERENCE (oracle/_ref/libmglp_ref.so, built from /root/reference/proj/src by
oracle/Makefile) on seeded synthetic inputs. Run in the build container:

    python tests/golden/make_golden.py

Inputs follow the reference's own generators: parameters from
LayerStack(cfg, seed) (blocks.cpp:432-449), z0 = 0.5*rng::gaussian(seed,
kTestOnly, 7, i) (tools/main.cpp:121-128) or testutil::random_tensor.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref as R  # noqa: E402

K_TEST = 6

CASES = {
    # name: stack, shape, solve
    "enc_small": dict(kind="encoder", d=16, heads=2, ffn=32, n_enc=8, n_dec=0, buffer_open=0,
                      buffer_close=0, seed=5, B=2, sx=6, sy=0, cf=2, levels=2, fwd_iters=2,
                      bwd_iters=1),
    "enc_small_3lvl": dict(kind="encoder", d=16, heads=4, ffn=24, n_enc=16, n_dec=0,
                           buffer_open=0, buffer_close=0, seed=11, B=2, sx=5, sy=0, cf=2,
                           levels=3, fwd_iters=3, bwd_iters=2),
    "causal_buffered": dict(kind="decoder_only", d=16, heads=2, ffn=32, n_enc=0, n_dec=10,
                            buffer_open=1, buffer_close=1, seed=6, B=2, sx=7, sy=0, cf=2,
                            levels=3, fwd_iters=2, bwd_iters=2),
    "encdec": dict(kind="encoder_decoder", d=16, heads=2, ffn=32, n_enc=4, n_dec=4,
                   buffer_open=0, buffer_close=0, seed=9, B=2, sx=5, sy=4, cf=2, levels=2,
                   fwd_iters=2, bwd_iters=1),
    # BASELINE.json configs[0]: the reference's CPU-runnable case
    "tiny_baseline": dict(kind="encoder", d=64, heads=2, ffn=256, n_enc=16, n_dec=0,
                          buffer_open=0, buffer_close=0, seed=7, B=8, sx=32, sy=0, cf=4,
                          levels=2, fwd_iters=1, bwd_iters=1, big=True),
}


def make(name, c):
    rc = R.RefStackConfig(kind=c["kind"], d=c["d"], heads=c["heads"], ffn=c["ffn"],
                          n_enc=c["n_enc"], n_dec=c["n_dec"], buffer_open=c["buffer_open"],
                          buffer_close=c["buffer_close"])
    st = R.RefStack(rc, c["seed"])
    B, sx, sy, d = c["B"], c["sx"], c["sy"], c["d"]
    n = B * (sx + sy) * d
    if c.get("big"):
        zx = R.gaussian_fill(c["seed"], K_TEST, 7, B * sx * d, 0.5)
        z0 = zx
        lam = R.gaussian_fill(8, K_TEST, 8, n, 1.0)
    else:
        z0 = R.gaussian_fill_flat(100 + c["seed"], K_TEST, n, 0.5)
        lam = R.gaussian_fill_flat(200 + c["seed"], K_TEST, n, 1.0)
    eng = R.RefEngine(st, coarsen=c["cf"], levels=c["levels"], fwd_iters=c["fwd_iters"],
                      bwd_iters=c["bwd_iters"], warm_start=False, workers=8)
    traj, ftr, fconv = eng.forward(z0, B, sx, sy)
    g = np.zeros(st.num_params())
    lam0, btr, bconv = eng.backward(traj, lam, B, sx, sy, grads=g)
    # serial reference for the same inputs
    straj = st.serial_forward(z0, B, sx, sy)
    sg = np.zeros(st.num_params())
    slam = st.serial_adjoint(straj, lam, B, sx, sy, grads=sg)
    params = st.get_params()
    meta = dict(c)
    meta["name"] = name
    meta["n_params"] = int(params.size)
    meta["params_sum"] = float(params.sum())
    meta["params_sumsq"] = float((params * params).sum())
    out = dict(meta=json.dumps(meta), z0=z0, lamN=lam, fwd_trace=np.array(ftr),
               bwd_trace=np.array(btr), lam0=lam0)
    if c.get("big"):
        total = traj.shape[0] - 1
        out.update(traj_last=traj[-1], traj_mid=traj[total // 2], serial_last=straj[-1],
                   serial_lam0=slam[0], grads_l2=np.array([np.linalg.norm(g)]),
                   grads_head=g[:4096].copy(), serial_grads_head=sg[:4096].copy(),
                   # every gradient entry (float32 is ample for a 1e-4 bar)
                   grads=g.astype(np.float32))
    else:
        out.update(params=params, traj=traj, grads=g, serial_traj=straj, serial_lam=slam,
                   serial_grads=sg)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {os.path.getsize(path) / 1024:.0f} KiB  fwd {ftr} bwd {btr}")


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for k in names:
        make(k, CASES[k])
