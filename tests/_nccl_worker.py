"""One rank of the multi-process NCCL parity test (tests/test_nccl_ranks.py),
launched by torchrun through tools/rank_one_gpu.sh: every rank on cuda:0,
NCCL's socket transport between the processes. Runs the distributed engine
(mglp_engine_create_dist: the real NcclTransport, not the loopback) for one
MGRIT fwd + bwd with gradients and saves this rank's owned trajectory
points, traces, lambda_0 and gradient block to <out>/rank<r>.npz.
Usage: bash tools/rank_one_gpu.sh tests/_nccl_worker.py <case-json> <out-dir>"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2601_09026_b200 import LayerStack, SolveConfig, StackConfig  # noqa: E402
from paper_2601_09026_b200 import _native as N  # noqa: E402
from paper_2601_09026_b200 import dist as D  # noqa: E402


def main():
    case = json.loads(sys.argv[1])
    out = sys.argv[2]
    rank, world = D.env_rank_world()
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")  # rendezvous + the NCCL id; the solve's traffic is NCCL
    sc = StackConfig(**case["stack"])
    so = SolveConfig(**case["solve"])
    params = np.ascontiguousarray(LayerStack(sc, 17).params(), np.float64)
    uid = D.share_unique_id(dist)
    h = D.create_engine(sc, so, 0, rank, world, uid)
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
    N.call("mglp_engine_backward_device", h, C.c_void_p(ld.data_ptr()), C.c_void_p(l0.data_ptr()), 1)
    N.call("mglp_engine_sync", h)
    info = [C.c_int() for _ in range(4)]
    N.call("mglp_engine_rank_info", h, *[C.byref(x) for x in info])
    total, ib = C.c_int(), C.c_int()
    N.call("mglp_engine_info", h, C.byref(total), C.byref(ib), None, None)
    lo, hi = info[2].value, info[3].value
    pts = list(range(ib.value + lo + 1, ib.value + hi + 1))
    if rank == world - 1:
        pts.append(total.value)  # the final state (closing buffers on the last rank)
    traj = np.empty((len(pts), ns.value), np.float32)
    for i, p in enumerate(pts):
        N.call("mglp_engine_read_traj", h, p, 1, traj[i].ctypes.data_as(C.POINTER(C.c_float)))
    g = np.zeros(params.size)
    N.call("mglp_engine_get_grads", h, N.dptr(g), g.size)
    tr = np.zeros(64)
    nt, cv = C.c_int(), C.c_int()
    N.call("mglp_engine_trace", h, 0, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
    ftr = tr[:nt.value].copy()
    N.call("mglp_engine_trace", h, 1, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
    btr = tr[:nt.value].copy()
    be, nr = C.c_int(), C.c_int()
    N.call("mglp_engine_comm_info", h, C.byref(be), C.byref(nr))
    np.savez(os.path.join(out, f"rank{rank}.npz"), pts=np.array(pts), traj=traj[:, :n],
             grads=g, ftr=ftr, btr=btr, l0=l0[:n].cpu().numpy(), backend=be.value,
             nranks=nr.value)
    N.call("mglp_engine_destroy", h)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
