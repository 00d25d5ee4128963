"""The multi-GPU path through the REAL NCCL transport, as separate processes:
P ranks launched by torchrun (tools/rank_one_gpu.sh: all on the one GPU a
test box has, NCCL's socket transport between the processes, per-rank
NCCL_HOSTID so NCCL accepts the shared device) run the distributed engine
(mglp_engine_create_dist, NcclTransport: ghost-exchange groups, the coarse
chain pipelined across ranks, all-gathered residual partials, broadcasts)
and must reproduce the single-rank solve BITWISE -- every rank's owned
states, both residual traces, lambda_0 and the gradients. (The in-process
loopback form of the same check: tests/test_dist.py.)"""
import ctypes as C
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2601_09026_b200 import LayerStack, SolveConfig, StackConfig
from paper_2601_09026_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [
    # d = 64, s = 128: the pre-split operand paths and the fused attention's pre-split P
    dict(stack=dict(kind="encoder", d=64, heads=2, ffn=128, n_enc=8),
         solve=dict(coarsen=2, levels=2, fwd_iters=2, bwd_iters=2, warm_start=False),
         B=1, sx=128, sy=0, worlds=[2, 4]),
    # three levels, the coarse chain two levels down
    dict(stack=dict(kind="encoder", d=16, heads=2, ffn=32, n_enc=16),
         solve=dict(coarsen=2, levels=3, fwd_iters=2, bwd_iters=2, warm_start=False),
         B=2, sx=6, sy=0, worlds=[2]),
    # causal decoder with open / close buffer layers on the edge ranks
    dict(stack=dict(kind="decoder_only", d=16, heads=2, ffn=32, n_dec=10, buffer_open=1,
                    buffer_close=1),
         solve=dict(coarsen=2, levels=2, fwd_iters=2, bwd_iters=2, warm_start=False),
         B=2, sx=6, sy=0, worlds=[2]),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _single_rank(case):
    import torch
    sc = StackConfig(**case["stack"])
    so = SolveConfig(**case["solve"])
    params = np.ascontiguousarray(LayerStack(sc, 17).params(), np.float64)
    h = C.c_void_p()
    N.call("mglp_engine_create", C.byref(sc.desc()), C.byref(so.desc()), 0, C.byref(h))
    try:
        B, sx, sy = case["B"], case["sx"], case["sy"]
        ns = C.c_longlong()
        N.call("mglp_engine_set_params", h, N.dptr(params), params.size)
        N.call("mglp_engine_set_shape", h, B, sx, sy, C.byref(ns))
        n = B * (sx + sy) * sc.d
        rng = np.random.default_rng(5)
        z0 = rng.standard_normal(n) * 0.5
        lam = rng.standard_normal(n)
        zd = torch.zeros(ns.value, device="cuda")
        ld = torch.zeros(ns.value, device="cuda")
        l0 = torch.zeros(ns.value, device="cuda")
        zd[:n] = torch.from_numpy(z0).float()
        ld[:n] = torch.from_numpy(lam).float()
        N.call("mglp_engine_zero_grads", h)
        N.call("mglp_engine_forward_device", h, C.c_void_p(zd.data_ptr()))
        N.call("mglp_engine_backward_device", h, C.c_void_p(ld.data_ptr()),
               C.c_void_p(l0.data_ptr()), 1)
        N.call("mglp_engine_sync", h)
        total = C.c_int()
        N.call("mglp_engine_info", h, C.byref(total), None, None, None)
        traj = np.empty((total.value + 1, ns.value), np.float32)
        N.call("mglp_engine_read_traj", h, 0, total.value + 1,
               traj.ctypes.data_as(C.POINTER(C.c_float)))
        g = np.zeros(params.size)
        N.call("mglp_engine_get_grads", h, N.dptr(g), g.size)
        tr = np.zeros(64)
        nt, cv = C.c_int(), C.c_int()
        N.call("mglp_engine_trace", h, 0, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
        ftr = tr[:nt.value].copy()
        N.call("mglp_engine_trace", h, 1, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
        btr = tr[:nt.value].copy()
        return dict(traj=traj[:, :n], grads=g, ftr=ftr, btr=btr, l0=l0[:n].cpu().numpy())
    finally:
        N.call("mglp_engine_destroy", h)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=["presplit_s128", "three_levels", "causal_buffers"])
def test_nccl_ranks_reproduce_single_rank_bitwise(case, tmp_path):
    ref = _single_rank(case)
    for world in case["worlds"]:
        out = tmp_path / f"w{world}"
        out.mkdir()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", "--no-python", "bash",
               os.path.join(ROOT, "tools", "rank_one_gpu.sh"),
               os.path.join(ROOT, "tests", "_nccl_worker.py"), json.dumps(case), str(out)]
        r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        gsum = np.zeros_like(ref["grads"])
        for rank in range(world):
            f = np.load(out / f"rank{rank}.npz")
            assert int(f["backend"]) == 1 and int(f["nranks"]) == world  # NCCL, P ranks
            pts = f["pts"]
            assert np.array_equal(f["traj"], ref["traj"][pts]), (world, rank)
            assert np.array_equal(f["ftr"], ref["ftr"]), (world, rank)
            assert np.array_equal(f["btr"], ref["btr"]), (world, rank)
            if rank == 0:
                assert np.array_equal(f["l0"], ref["l0"]), world
            gsum += f["grads"]
        assert np.array_equal(gsum, ref["grads"]), world
