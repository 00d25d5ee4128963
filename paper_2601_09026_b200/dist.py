"""Multi-GPU plumbing for the layer-parallel engine.

One process per GPU. torch.distributed is used only for the rendezvous and to
share NCCL's 128-byte unique id; all solver traffic goes through NCCL inside
libmglp_cuda.so (send/recv of boundary states over NVLink).

`owned_points` restates the engine's partition (engine.cu alloc_solver) so
hosts can reason about which rank holds what without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _native as N
from .engine import SolveConfig, StackConfig, ValidationError


def level_sizes(n_steps: int, cf: int, levels: int):
    n = [n_steps]
    for _ in range(1, max(levels, 2)):
        n.append(n[-1] // cf)
    return n


def check_partition(n_steps: int, cf: int, levels: int, world: int):
    """ValidationError unless every level's coarse intervals split evenly."""
    n = n_steps
    for l in range(max(levels, 2) - 1):
        if (n // cf) % world:
            raise ValidationError(f"layer partition: the {n // cf} coarse intervals of level {l} "
                                  f"do not split over {world} ranks")
        n //= cf
        if l + 2 >= levels:
            break


def owned_points(n_steps: int, cf: int, levels: int, rank: int, world: int, adjoint=False):
    """Per level, the (p_lo, p_hi] points this rank owns (p_lo is a ghost)."""
    check_partition(n_steps, cf, levels, world)
    tpos = world - 1 - rank if adjoint else rank
    return [(tpos * (n // world), (tpos + 1) * (n // world)) for n in level_sizes(n_steps, cf, levels)]


def owned_layers(n_steps: int, cf: int, levels: int, rank: int, world: int):
    lo, hi = owned_points(n_steps, cf, levels, rank, world)[0]
    return lo, hi


def env_rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def share_unique_id(dist, device=None) -> bytes:
    """Rank 0 creates NCCL's unique id; every rank returns the same 128 bytes."""
    import torch
    rank = dist.get_rank()
    buf = (C.c_char * 128)()
    if rank == 0:
        N.call("mglp_nccl_unique_id", C.cast(buf, C.c_void_p))
    backend = dist.get_backend()
    dev = device if (backend == "nccl" and device is not None) else "cpu"
    t = torch.tensor(list(bytes(buf)), dtype=torch.uint8, device=dev)
    dist.broadcast(t, src=0)
    return bytes(t.cpu().tolist())


def create_engine(stack: StackConfig, solve: SolveConfig, device: int, rank: int, world: int,
                  uid: bytes):
    """mglp_engine_create_dist: this rank's block of the layer-parallel engine."""
    h = C.c_void_p()
    idbuf = (C.c_char * 128).from_buffer_copy(uid) if uid is not None else None
    N.call("mglp_engine_create_dist", C.byref(stack.desc()), C.byref(solve.desc()), device, rank,
           world, C.cast(idbuf, C.c_void_p) if idbuf is not None else None, C.byref(h))
    return h
