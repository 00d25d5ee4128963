"""Kernel-variant switches that must not change a single bit of the solve:
the pair GEMM's TMEM-drain epilogue (MGLP_GEMM_DRAIN=0 vs the default), the
s = 128 attention backward's alternating dO / V regions
(MGLP_ATTN_PINGPONG=0) and the head-split pre-split attention operands
(MGLP_NO_ATTN_HS=1: the kernels split fp32 operands themselves -- the same
split arithmetic, so the same tiles). Each setting runs in its own process
(the switches are read once per process) on a stack wide enough for the
CTA-pair GEMM (M, N >= 256) at s = 128."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %(root)r)
from paper_2601_09026_b200 import LayerParallelEngine, LayerStack, SolveConfig, StackConfig, State
d, H, f, L, B, s = 256, 4, 1024, 8, 4, 128
st = LayerStack(StackConfig(kind=%(kind)r, d=d, heads=H, ffn=f, n_enc=L if %(kind)r == "encoder" else 0,
                            n_dec=L if %(kind)r != "encoder" else 0), 5, device=0)
eng = LayerParallelEngine(st, SolveConfig(coarsen=2, levels=2, fwd_iters=1, bwd_iters=1,
                                          warm_start=False))
rng = np.random.default_rng(3)
z0 = State.from_flat(rng.standard_normal(B * s * d) * 0.5, B, s, 0, d)
lam = State.from_flat(rng.standard_normal(B * s * d), B, s, 0, d)
fo = eng.forward(z0)
g = st.zero_grads()
bo = eng.backward(fo.traj, lam, g)
np.savez(%(out)r, traj=np.stack([t.flat() for t in fo.traj]), lam0=bo.lambda0.flat(),
         grads=np.asarray(g), ft=np.asarray(fo.phase.trace), bt=np.asarray(bo.phase.trace))
"""


def run(tmp_path, kind, env):
    out = str(tmp_path / f"{kind}_{abs(hash(json.dumps(env, sort_keys=True)))}.npz")
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT, "kind": kind, "out": out}],
                   check=True, env=e, timeout=600)
    return np.load(out)


@pytest.mark.parametrize("kind", ["encoder", "decoder_only"])
@pytest.mark.parametrize("env", [{"MGLP_GEMM_DRAIN": "0"}, {"MGLP_ATTN_PINGPONG": "0"},
                                 {"MGLP_NO_ATTN_HS": "1"}])
def test_variant_is_bitwise_the_default(tmp_path, kind, env):
    a = run(tmp_path, kind, {})
    b = run(tmp_path, kind, env)
    for k in ("traj", "lam0", "grads", "ft", "bt"):
        assert np.array_equal(a[k], b[k]), (env, k)
