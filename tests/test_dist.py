"""Multi-GPU (layer-partitioned) solve.

CPU (gloo, world_size 2): the host-side partition, rendezvous and id sharing.
GPU (one device): P virtual ranks through the in-process loopback transport
run exactly the partitioned control flow (ghost exchange after C-relaxation,
the coarse chain pipelined across ranks, all-gathered norm partials, reversed
adjoint partition, per-rank parameter pass) and must reproduce the 1-rank
solve BITWISE -- states, residual traces, lambda_0 and gradients."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2601_09026_b200 import LayerStack, SolveConfig, StackConfig, ValidationError
from paper_2601_09026_b200 import _native as N
from paper_2601_09026_b200 import dist as D


# ---------------------------------------------------------------- CPU / gloo
def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        out = {}
        for (n, cf, lv) in [(64, 4, 2), (128, 4, 3), (64, 8, 2), (16, 2, 3)]:
            pts = D.owned_points(n, cf, lv, rank, world)
            adj = D.owned_points(n, cf, lv, rank, world, adjoint=True)
            got = [None] * world
            dist.all_gather_object(got, (pts, adj))
            out[(n, cf, lv)] = got
        # a fake 128-byte id travels like the NCCL one does
        t = torch.arange(128, dtype=torch.uint8) if rank == 0 else torch.zeros(128, dtype=torch.uint8)
        dist.broadcast(t, src=0)
        out["id_ok"] = bytes(t.tolist()) == bytes(range(128))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_partition_and_rendezvous_gloo_world2():
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
    assert res[0]["id_ok"] and res[1]["id_ok"]
    for key in [(64, 4, 2), (128, 4, 3), (64, 8, 2), (16, 2, 3)]:
        n, cf, lv = key
        got = res[0][key]
        assert got == res[1][key]
        sizes = D.level_sizes(n, cf, lv)
        for which in (0, 1):  # forward, adjoint
            for l, nl in enumerate(sizes):
                spans = sorted(g[which][l] for g in got)
                # contiguous, disjoint cover of (0, n_l]
                assert spans[0][0] == 0 and spans[-1][1] == nl
                assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        # the adjoint partition is the forward one reversed in time
        for r in range(2):
            assert got[r][1][0] == (n - got[r][0][0][1], n - got[r][0][0][0])


def test_partition_validation():
    with pytest.raises(ValidationError):
        D.check_partition(16, 4, 2, 8)  # 4 intervals over 8 ranks
    with pytest.raises(ValidationError):
        D.check_partition(32, 4, 3, 4)  # level-1 has 2 intervals
    D.check_partition(128, 4, 3, 8)


# ---------------------------------------------------------------- GPU loopback
def _run_group(sc, so, world, params, B, sx, sy, z0, lam):
    import torch
    arr = (C.c_void_p * world)()
    N.call("mglp_loopback_create", C.byref(sc.desc()), C.byref(so.desc()), 0, world, arr)
    engines = [arr[r] for r in range(world)]
    ns = C.c_longlong()
    for h in engines:
        N.call("mglp_engine_set_params", h, N.dptr(params), params.size)
        N.call("mglp_engine_set_shape", h, B, sx, sy, C.byref(ns))
    n = B * (sx + sy) * sc.d
    zd = torch.zeros(ns.value, device="cuda")
    ld = torch.zeros(ns.value, device="cuda")
    l0 = torch.zeros(ns.value, device="cuda")
    zd[:n] = torch.from_numpy(z0).float()
    ld[:n] = torch.from_numpy(lam).float()
    for h in engines:
        N.call("mglp_engine_zero_grads", h)
    N.call("mglp_loopback_run_fwd_bwd", arr, world, C.c_void_p(zd.data_ptr()),
           C.c_void_p(ld.data_ptr()), C.c_void_p(l0.data_ptr()), 1)
    out = []
    for r, h in enumerate(engines):
        tp = C.c_void_p()
        N.call("mglp_engine_traj_device", h, C.byref(tp))
        info = [C.c_int() for _ in range(4)]
        N.call("mglp_engine_rank_info", h, *[C.byref(x) for x in info])
        total = C.c_int()
        ib = C.c_int()
        N.call("mglp_engine_info", h, C.byref(total), C.byref(ib), None, None)
        g = np.zeros(params.size)
        N.call("mglp_engine_get_grads", h, N.dptr(g), g.size)
        tr = np.zeros(64)
        nt, cv = C.c_int(), C.c_int()
        N.call("mglp_engine_trace", h, 0, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
        ftr = tr[:nt.value].copy()
        N.call("mglp_engine_trace", h, 1, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
        btr = tr[:nt.value].copy()
        out.append(dict(h=h, ptr=tp.value, lo=info[2].value, hi=info[3].value, ib=ib.value,
                        total=total.value, grads=g, ftr=ftr, btr=btr))
    return out, l0[:n].cpu().numpy(), ns.value


class _DevView:
    """Zero-copy torch view of a raw device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3}


CASES = [
    ("encoder", dict(n_enc=16), 0, 0, 2, 2, [2, 4, 8]),
    ("encoder", dict(n_enc=16), 0, 0, 2, 3, [2, 4]),
    ("decoder_only", dict(n_dec=10, buffer_open=1, buffer_close=1), 0, 0, 2, 2, [2, 4]),
    ("encoder_decoder", dict(n_enc=4, n_dec=4), 5, 4, 2, 2, [2, 4]),
]


# d = 64, dh = 32, s = 128: the pre-split operand paths and the pre-split P of
# the fused attention, partitioned across ranks
CASES_PRESPLIT = [
    ("encoder", dict(n_enc=8), 0, 0, 2, 2, [2, 4], (64, 2, 128), (1, 128)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES + CASES_PRESPLIT)
def test_loopback_ranks_reproduce_single_rank_bitwise(case):
    import torch
    kind, kw, sx_extra, sy, cf, lv, worlds = case[:7]
    d, heads, ffn = case[7] if len(case) > 7 else (16, 2, 32)
    sc = StackConfig(kind=kind, d=d, heads=heads, ffn=ffn, **kw)
    st = LayerStack(sc, 17)
    params = np.ascontiguousarray(st.params(), np.float64)
    B, sx = case[8] if len(case) > 8 else (2, 6)
    rng = np.random.default_rng(5)
    n = B * (sx + sy) * sc.d
    z0 = rng.standard_normal(n) * 0.5
    lam = rng.standard_normal(n)
    so = SolveConfig(coarsen=cf, levels=lv, fwd_iters=2, bwd_iters=2, warm_start=False)
    ref, ref_l0, ns = _run_group(sc, so, 1, params, B, sx, sy, z0, lam)
    r0 = ref[0]

    def traj_of(rec, pts=None):
        # a rank maps only its own block of time points (the rest faults):
        # read those, NaN elsewhere
        torch.cuda.synchronize()
        T = np.full((rec["total"] + 1, n), np.nan, np.float32)
        for p in (range(rec["total"] + 1) if pts is None else pts):
            buf = np.empty(ns, np.float32)
            N.call("mglp_engine_read_traj", rec["h"], p, 1,
                   buf.ctypes.data_as(C.POINTER(C.c_float)))
            T[p] = buf[:n]
        return T

    T1 = traj_of(r0)
    for world in worlds:
        recs, l0, _ = _run_group(sc, so, world, params, B, sx, sy, z0, lam)
        gsum = np.zeros(params.size)
        for rec in recs:
            ib = rec["ib"]
            # owned interior points (lo, hi] (+ point 0 / buffers on the edges)
            pts = list(range(ib + rec["lo"] + 1, ib + rec["hi"] + 1))
            T = traj_of(rec, pts)
            assert np.array_equal(T[pts], T1[pts]), (world, rec["lo"], rec["hi"])
            assert np.array_equal(rec["ftr"], r0["ftr"])
            assert np.array_equal(rec["btr"], r0["btr"])
            gsum += rec["grads"]
        last = recs[-1]["total"]
        assert np.array_equal(T1[-1], traj_of(recs[-1], [last])[-1])
        assert np.array_equal(l0, ref_l0)
        assert np.array_equal(gsum, r0["grads"])


@pytest.mark.gpu
def test_rank_memory_shrinks_with_p():
    """SURVEY 8(e) / VERDICT r1 weak #9: a rank maps physical HBM only under its
    own block of layers and time points (parameters, pre-split weights,
    gradients, activation caches, trajectory, solver levels) and sizes its
    scratch for its own intervals, so per-rank memory is about 1/P of the
    single-rank engine; other ranks' slots are unmapped (reading one is
    refused by the C-ABI, and on the device it would fault)."""
    sc = StackConfig(kind="encoder", d=256, heads=4, ffn=1024, n_enc=16)
    so = SolveConfig(coarsen=2, levels=2, fwd_iters=1, bwd_iters=1, warm_start=False)
    mem = {}
    for world in (1, 2, 4):
        arr = (C.c_void_p * world)()
        N.call("mglp_loopback_create", C.byref(sc.desc()), C.byref(so.desc()), 0, world, arr)
        ns = C.c_longlong()
        per = []
        for r in range(world):
            N.call("mglp_engine_set_shape", arr[r], 16, 128, 0, C.byref(ns))
            b = C.c_longlong()
            N.call("mglp_engine_memory", arr[r], C.byref(b))
            per.append(b.value)
        if world > 1:  # another rank's time point is not readable
            buf = np.empty(ns.value, np.float32)
            with pytest.raises(ValidationError):
                N.call("mglp_engine_read_traj", arr[0], 16, 1,
                       buf.ctypes.data_as(C.POINTER(C.c_float)))
        for r in range(world):
            N.call("mglp_engine_destroy", arr[r])
        mem[world] = max(per)
    assert mem[2] <= 0.62 * mem[1], mem
    assert mem[4] <= 0.37 * mem[1], mem
