#!/usr/bin/env python
"""Device-timed MGRIT fwd+bwd iteration on B200 (BASELINE.json metric).

One step = one layer-parallel training-step solve of the hot path:
LayerParallelEngine::forward (k_f V-cycles of forward MGRIT) + ::backward
(k_b cycles of adjoint MGRIT + the parameter-gradient pass), cold broadcast
guess every step (warm start off, so every step does identical work;
SURVEY 8(d)). Workload = BASELINE configs[1] (BERT-base-style ODE encoder,
L=64, d=768, 12 heads, seq 128, batch 32, 2-level MGRIT c_f=4, 1+1 cycles)
unless --config says otherwise. Synthetic inputs: parameters from
LayerStack(cfg, seed=7) (reference init, bit-identical), z0 =
0.5*rng::gaussian(7, kTestOnly, 7, i), lambda_N = rng::gaussian(8, kTestOnly, 8, i).

Also measured: the device serial fwd+bwd (serial_forward + serial_adjoint with
gradients) for the speedup; a profiled step for the roofline of the dominant
kernel (tcgen05 GEMM); an end-to-end step through the public API with
pinned-host inputs; and (rank 0, N=1) the reference CPU implementation on a
bounded sample. `--impl reference` prints the reference arm instead.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "tiny": dict(desc="tiny ODE-transformer encoder L=16 d=64 2 heads seq 32 batch 8, 2-level cf=4",
                 kind="encoder", n_enc=16, n_dec=0, d=64, H=2, ffn=256, sx=32, sy=0, B=8, cf=4,
                 levels=2, fwd=1, bwd=1),
    "bert": dict(desc="BERT-base-style ODE encoder L=64 d=768 seq 128 batch 32, 2-level MGRIT cf=4",
                 kind="encoder", n_enc=64, n_dec=0, d=768, H=12, ffn=3072, sx=128, sy=0, B=32,
                 cf=4, levels=2, fwd=1, bwd=1),
    "gpt": dict(desc="GPT-2-small-style causal ODE decoder L=128 d=768 seq 512 batch 8, 3-level cf=4",
                kind="decoder_only", n_enc=0, n_dec=128, d=768, H=12, ffn=3072, sx=512, sy=0, B=8,
                cf=4, levels=3, fwd=1, bwd=1),
    "vit": dict(desc="ViT-B/16-style ODE encoder L=64 d=768 197 tokens batch 32, 2-level cf=8",
                kind="encoder", n_enc=64, n_dec=0, d=768, H=12, ffn=3072, sx=197, sy=0, B=32,
                cf=8, levels=2, fwd=1, bwd=1),
    "mt": dict(desc="encoder-decoder ODE transformer L=32+32 d=512 seq 128 batch 32, 2-level cf=4",
               kind="encoder_decoder", n_enc=32, n_dec=32, d=512, H=8, ffn=2048, sx=128, sy=128,
               B=32, cf=4, levels=2, fwd=1, bwd=1),
}
METRIC = "MGRIT fwd+bwd iteration time & speedup vs serial, 1/2/4/8 B200"
K_TEST = 6  # rng::kTestOnly


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference CPU implementation (oracle/_ref = the unmodified reference sources)
# ---------------------------------------------------------------------------
def mgrit_critical_path(N, cf, levels, P):
    """Reference-executor critical path of one V-cycle, in serial Phi units,
    with P workers (Executor::run over chunk tasks, mgrit.hpp:125-246)."""
    def ceil(a, b):
        return -(-a // b)
    n = [N]
    for _ in range(1, max(levels, 2)):
        n.append(n[-1] // cf)

    def fcf(l):
        nc = n[l] // cf
        return 2 * ceil(nc, P) * (cf - 1) + ceil(nc, P)

    def resid(l):
        return ceil(n[l] // cf, P) * cf

    def descend(l):
        if l == levels - 1:
            return n[l]  # serial exact solve
        return (fcf(l) + resid(l) + ceil(n[l + 1], P) + descend(l + 1)
                + ceil(n[l] // cf, P) * (cf - 1))

    t = fcf(0) + resid(0)
    if levels > 1:
        t += ceil(n[1], P) + descend(1) + ceil(n[0] // cf, P) * (cf - 1)
    return t


def reference_sample(cfg, workers):
    """Times the compiled reference's LayerStack::step and ::adjoint_step (with
    grads) at batch 1 on the config's block shape, `workers` of them running
    concurrently on distinct layers (one host thread each -- what the
    reference Executor does with its chunk tasks, memory contention included),
    and extrapolates one MGRIT fwd+bwd iteration (ms) at the config's batch
    from the Executor's critical path in such rounds of `workers` Phi."""
    import threading

    import numpy as np
    from oracle import ref as R
    kind = cfg["kind"]
    P = workers
    rc = R.RefStackConfig(kind=kind, d=cfg["d"], heads=cfg["H"], ffn=cfg["ffn"])
    if kind == "encoder":
        rc.n_enc, rc.n_dec = P, 0
    elif kind == "decoder_only":
        rc.n_enc, rc.n_dec = 0, P
    else:  # half encoder, half decoder layers in every round
        rc.n_enc, rc.n_dec = (P + 1) // 2, max(1, P // 2)
    st = R.RefStack(rc, 7)
    d, sx, sy = cfg["d"], cfg["sx"], cfg["sy"]
    n = (sx + sy) * d
    z = R.gaussian_fill(7, K_TEST, 7, n, 0.5)
    lam = R.gaussian_fill(8, K_TEST, 8, n, 1.0)
    g = np.zeros(st.num_params())
    layers = list(range(st.total))[:P]

    def concurrent(fn):
        ts = [threading.Thread(target=fn, args=(layer,)) for layer in layers]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return time.perf_counter() - t0

    def one(fn):
        t0 = time.perf_counter()
        fn(layers[0])
        return time.perf_counter() - t0

    step = lambda layer: st.step(layer, 1.0, z, 1, sx, sy)  # noqa: E731
    adj = lambda layer: st.adjoint_step(layer, 1.0, z, lam, 1, sx, sy, grads=g,  # noqa: E731
                                        gscale=1.0)
    # ctypes releases the GIL for the duration of each reference call
    t_step, t_adj = concurrent(step), concurrent(adj)
    t1_step, t1_adj = one(step), one(adj)
    N = cfg["n_enc"] + cfg["n_dec"]
    cp = mgrit_critical_path(N, cfg["cf"], cfg["levels"], P)
    B = cfg["B"]
    # forward: k_f cycles; backward: k_b cycles + parameter pass (N tasks).
    # The reference's adjoint_step always forms dW (tensor.cpp:220-237), so a
    # Phi^T without gradients costs the same as one with.
    fwd = cfg["fwd"] * cp * t_step * B
    bwd = (cfg["bwd"] * cp + -(-N // P)) * t_adj * B
    serial = N * (t1_step + t1_adj) * B  # one thread, layer after layer
    return {"ms": (fwd + bwd) * 1e3, "serial_ms": serial * 1e3, "t_step_s": t_step,
            "t_adjoint_step_s": t_adj, "threads": P,
            "sample": (f"{P} concurrent LayerStack::step and {P} concurrent ::adjoint_step(grads) "
                       f"(one host thread per layer, compiled reference oracle/_ref) at batch 1 "
                       f"on the config's block shape; extrapolated to one MGRIT "
                       f"{cfg['fwd']}+{cfg['bwd']} iteration at batch {B}: {cp} rounds of {P} Phi "
                       f"per cycle on the reference Executor's critical path (round t_step="
                       f"{t_step:.3g}s, t_adj={t_adj:.3g}s)")}


def run_reference_arm(args, cfg, rank, world):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference sources) on the host cores, on this arm's config and metric.
    tiny (configs[0]) runs in full: LayerParallelEngine::forward + ::backward
    with Executor(cores) (adjoint.hpp:113-183, executor.cpp:75-121). The large
    configs take hours per iteration on the CPU, so each step is the bounded
    per-layer sample of reference_sample(), extrapolated -- and the line
    carries the same model evaluated on tiny next to tiny's full measurement,
    the extrapolation's measured error."""
    if rank != 0:
        return
    from oracle import ref as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libmglp_ref.so not built (needs /root/reference at build)"}))
        return
    threads = max(1, min(os.cpu_count() or 1, cfg["n_enc"] + cfg["n_dec"]))
    full = args.config == "tiny"
    samples = []
    for i in range(args.warmup + args.steps):
        s = reference_full(cfg, threads) if full else reference_sample(cfg, threads)
        if i >= args.warmup:
            samples.append(s)
    ms = statistics.median(s["ms"] for s in samples)
    s0 = samples[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms/iteration",
        "higher_is_better": False, "n_gpus": world if world > 1 else args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference LayerStack init seed 7; z0/lambda_N from rng::gaussian)",
        "config": config_block(args.config, cfg, 1),
        "serial_ms": statistics.median(s["serial_ms"] for s in samples),
        "measured_in_full": full,
        "cpu_baseline": {"value": ms, "unit": "ms/iteration", "cores": threads,
                         "kind": "reference", "sample": s0["sample"]},
        "e2e": {"value": ms, "unit": "ms/iteration", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if not full:
        line["extrapolation_check"] = extrapolation_check()
    print(json.dumps(line), flush=True)


def reference_full(cfg, workers):
    """One full MGRIT fwd+bwd iteration of the compiled reference engine with
    Executor(workers), and its serial fwd+bwd (one thread) -- tiny only."""
    import numpy as np
    from oracle import ref as R
    rc = R.RefStackConfig(kind=cfg["kind"], d=cfg["d"], heads=cfg["H"], ffn=cfg["ffn"],
                          n_enc=cfg["n_enc"], n_dec=cfg["n_dec"])
    st = R.RefStack(rc, 7)
    B, sx, sy, d = cfg["B"], cfg["sx"], cfg["sy"], cfg["d"]
    n = B * (sx + sy) * d
    z0 = R.gaussian_fill(7, K_TEST, 7, n, 0.5)
    lam = R.gaussian_fill(8, K_TEST, 8, n, 1.0)
    eng = R.RefEngine(st, coarsen=cfg["cf"], levels=cfg["levels"], fwd_iters=cfg["fwd"],
                      bwd_iters=cfg["bwd"], warm_start=False, workers=workers)
    g = np.zeros(st.num_params())
    t0 = time.perf_counter()
    traj, _, _ = eng.forward(z0, B, sx, sy)
    eng.backward(traj, lam, B, sx, sy, grads=g)
    t1 = time.perf_counter()
    tr = st.serial_forward(z0, B, sx, sy)
    st.serial_adjoint(tr, lam, B, sx, sy, grads=g)
    t2 = time.perf_counter()
    return {"ms": (t1 - t0) * 1e3, "serial_ms": (t2 - t1) * 1e3,
            "sample": (f"the full iteration: compiled reference LayerParallelEngine forward + "
                       f"backward (grads) with Executor({workers}) at batch {B}, "
                       f"{cfg['fwd']}+{cfg['bwd']} cycles; serial_forward + serial_adjoint on one "
                       f"thread")}


def extrapolation_check():
    """reference_sample's per-layer model against a full reference run, on tiny"""
    cfg = CONFIGS["tiny"]
    threads = max(1, min(os.cpu_count() or 1, cfg["n_enc"] + cfg["n_dec"]))
    full = min((reference_full(cfg, threads) for _ in range(3)), key=lambda s: s["ms"])
    model = min((reference_sample(cfg, threads) for _ in range(3)), key=lambda s: s["ms"])
    return {"config": "tiny", "measured_ms": full["ms"], "modelled_ms": model["ms"],
            "model_error": model["ms"] / full["ms"] - 1.0,
            "measured_serial_ms": full["serial_ms"], "modelled_serial_ms": model["serial_ms"],
            "serial_model_error": model["serial_ms"] / full["serial_ms"] - 1.0}


# ---------------------------------------------------------------------------
# device arm
# ---------------------------------------------------------------------------
def gemm_flops_per_iteration(cfg):
    """Algorithmic FLOPs of one layer evaluation: linear, attention."""
    d, f, B = cfg["d"], cfg["ffn"], cfg["B"]
    T = B * cfg["sx"]
    s = cfg["sx"]
    causal = cfg["kind"] == "decoder_only"
    lin = 2 * T * (4 * d * d + 2 * d * f)
    att = 4 * B * s * s * d * (0.5 if causal else 1.0)
    return lin, att


def config_block(name, cfg, world):
    n = cfg["n_enc"] + cfg["n_dec"]
    return {"workload": name, "desc": cfg["desc"],
            "hierarchy": f"cf={cfg['cf']} levels={cfg['levels']} fwd={cfg['fwd']} "
                         f"bwd={cfg['bwd']} cold broadcast guess",
            "parallelism": f"layer-parallel x{world} (contiguous blocks of {n // world} layers "
                           f"per GPU; boundary states over NCCL send/recv)",
            "l2": "inputs > L2: states + activation cache are GBs (>> 126 MB L2)",
            "gemm_precision": "tcgen05 kind::f16 3-pass split (hi + 2^-11 lo', ~22-bit operands), "
                              "fp32 accumulate"}


def traffic_evidence():
    """DRAM bytes per launch of the dominant kernel from the newest committed
    ncu --set full capture (profiles/r*_ncu_traffic.json)"""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_traffic.json")))
    if not files:
        return None, None
    tj = json.load(open(files[-1]))
    return tj["traffic_bytes_per_launch"], tj["source"]


class DeviceRun:
    """One config's engine on this rank (one process per GPU; N > 1: this
    rank's block of layers, NCCL inside the library)."""

    def __init__(self, name, args, rank, world, dist, local):
        import numpy as np
        import torch
        from paper_2601_09026_b200 import _native as N
        from paper_2601_09026_b200.engine import SolveConfig, StackConfig
        self.N, self.np, self.torch = N, np, torch
        self.name, self.cfg, self.args = name, CONFIGS[name], args
        self.rank, self.world, self.dist, self.local = rank, world, dist, local
        cfg = self.cfg
        self.sc = StackConfig(kind=cfg["kind"], d=cfg["d"], heads=cfg["H"], ffn=cfg["ffn"],
                              n_enc=cfg["n_enc"], n_dec=cfg["n_dec"])
        self.so = SolveConfig(coarsen=cfg["cf"], levels=cfg["levels"], fwd_iters=cfg["fwd"],
                              bwd_iters=cfg["bwd"], warm_start=False)
        self.dev = torch.device("cuda", local)
        self.h = self._create(world)
        N.call("mglp_engine_init_params", self.h, C.c_ulonglong(7), None)
        ns = C.c_longlong()
        N.call("mglp_engine_set_shape", self.h, cfg["B"], cfg["sx"], cfg["sy"], C.byref(ns))
        self.n_state = ns.value
        self.n_logical = cfg["B"] * (cfg["sx"] + cfg["sy"]) * cfg["d"]
        self.z0h = np.empty(self.n_logical)
        N.call("mglp_rng_gaussian_fill", 7, K_TEST, 7, 0.5, N.dptr(self.z0h), self.n_logical)
        self.lamh = np.empty(self.n_logical)
        N.call("mglp_rng_gaussian_fill", 8, K_TEST, 8, 1.0, N.dptr(self.lamh), self.n_logical)
        self.z0 = torch.zeros(self.n_state, dtype=torch.float32, device=self.dev)
        self.lam = torch.zeros_like(self.z0)
        self.lam0 = torch.zeros_like(self.z0)
        self.z0[:self.n_logical] = torch.from_numpy(self.z0h).float()
        self.lam[:self.n_logical] = torch.from_numpy(self.lamh).float()
        sp = C.c_void_p()
        N.call("mglp_engine_stream", self.h, C.byref(sp))
        self.stream = torch.cuda.ExternalStream(sp.value, device=self.dev)
        self.graph = False
        torch.cuda.synchronize()

    def _create(self, world):
        N = self.N
        h = C.c_void_p()
        if world > 1:
            from paper_2601_09026_b200 import dist as D
            uid = D.share_unique_id(self.dist, device=self.dev)
            h = D.create_engine(self.sc, self.so, self.local, self.rank, world, uid)
        else:
            N.call("mglp_engine_create", C.byref(self.sc.desc()), C.byref(self.so.desc()),
                   self.local, C.byref(h))
        return h

    def close(self):
        if self.h is not None:
            self.N.call("mglp_engine_destroy", self.h)
            self.h = None
        self.torch.cuda.synchronize()

    # ---- steps ----
    def eager_step(self):
        N = self.N
        N.call("mglp_engine_forward_device", self.h, C.c_void_p(self.z0.data_ptr()))
        N.call("mglp_engine_backward_device", self.h, C.c_void_p(self.lam.data_ptr()),
               C.c_void_p(self.lam0.data_ptr()), 1)

    def step(self):
        if self.graph:
            self.N.call("mglp_engine_graph_replay", self.h)
        else:
            self.eager_step()

    def serial_step(self):
        N = self.N
        N.call("mglp_serial_forward_device", self.h, C.c_void_p(self.z0.data_ptr()))
        N.call("mglp_serial_adjoint_device", self.h, C.c_void_p(self.lam.data_ptr()),
               C.c_void_p(self.lam0.data_ptr()), 1)

    def capture(self):
        """the whole step (both solves, with N > 1 the NCCL exchanges NCCL
        records into the graph) as one CUDA graph launch"""
        N = self.N
        try:
            N.call("mglp_engine_graph_capture", self.h, C.c_void_p(self.z0.data_ptr()),
                   C.c_void_p(self.lam.data_ptr()), C.c_void_p(self.lam0.data_ptr()), 1)
            self.graph = True
            for _ in range(2):
                self.step()
            N.call("mglp_engine_sync", self.h)
            return None
        except Exception as ex:  # noqa: BLE001 -- reported in the JSON line
            self.graph = False
            N.call("mglp_engine_sync", self.h)
            return f"graph capture failed, eager: {ex}"

    def device_timed(self, fn, k):
        """k calls of fn, CUDA events on the engine stream, barrier + sync on
        both sides, max over ranks"""
        torch = self.torch
        if self.dist is not None:
            self.dist.barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(self.stream)
        for _ in range(k):
            fn()
        b.record(self.stream)
        torch.cuda.synchronize()
        self.N.call("mglp_engine_sync", self.h)
        return self.max_over_ranks(a.elapsed_time(b) / k)

    def max_over_ranks(self, v):
        if self.dist is None:
            return v
        t = self.torch.tensor([v], device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def traces(self):
        N, np = self.N, self.np
        tr = np.empty(64)
        nt, cv = C.c_int(), C.c_int()
        N.call("mglp_engine_trace", self.h, 0, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
        f = list(tr[:nt.value])
        N.call("mglp_engine_trace", self.h, 1, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
        return f, list(tr[:nt.value])

    def launches(self):
        cnt = C.c_longlong()
        self.N.call("mglp_engine_take_launch_count", self.h, C.byref(cnt))
        return cnt.value

    def comm_info(self):
        b, n = C.c_int(), C.c_int()
        self.N.call("mglp_engine_comm_info", self.h, C.byref(b), C.byref(n))
        return {0: "none", 1: "nccl", 2: "loopback"}[b.value], n.value

    def probe_ms(self):
        """monitor probe step (controller.hpp:88-105 ProbeScope: both budgets
        doubled for one batch), eager; the captured step is re-captured after"""
        N = self.N
        sdesc = N.SolveDesc()
        N.call("mglp_engine_get_config", self.h, C.byref(sdesc))
        f0, b0 = sdesc.fwd_iters, sdesc.bwd_iters
        sdesc.fwd_iters, sdesc.bwd_iters = 2 * f0, 2 * b0
        N.call("mglp_engine_set_config", self.h, C.byref(sdesc))
        self.eager_step()
        ms = self.device_timed(self.eager_step, 1)
        sdesc.fwd_iters, sdesc.bwd_iters = f0, b0
        N.call("mglp_engine_set_config", self.h, C.byref(sdesc))
        if self.graph:
            self.capture()
        return ms, f"fwd={2 * f0} bwd={2 * b0} (ProbeScope doubling, eager launch)"

    def profile(self):
        """per-kernel-class device time of one eager step (CUDA events around
        every launch, outside any timed region)"""
        N = self.N
        N.call("mglp_engine_profile", self.h, 1)
        self.eager_step()
        ms3, fl3, by3 = (C.c_double * 3)(), (C.c_double * 3)(), (C.c_double * 3)()
        ln3 = (C.c_longlong * 3)()
        N.call("mglp_engine_profile_read", self.h, ms3, fl3, by3, ln3)
        N.call("mglp_engine_profile", self.h, 0)
        return list(ms3), list(fl3), list(by3), list(ln3)

    def e2e(self, k):
        """The reference-facing C-ABI with HOST buffers every step:
        mglp_engine_forward(z0 f64) + mglp_engine_backward_keep_grads(lambda_N
        f64 -> lambda_0 f64), i.e. CudaLayerParallelEngine::forward/backward
         with the gradients left in the device slab for the
        device optimizer; f64 -> fp32 conversion, pinned H2D, the solve, D2H of
        lambda_0 and both traces inside the timed region (wall clock, max
        over ranks)."""
        N, np, torch = self.N, self.np, self.torch
        cfg = self.cfg
        lam0 = np.empty(self.n_logical)
        tr = np.empty(64)
        nt, cv = C.c_int(), C.c_int()

        def one():
            N.call("mglp_engine_forward", self.h, cfg["B"], cfg["sx"], cfg["sy"],
                   N.dptr(self.z0h), None, N.dptr(tr), 64, C.byref(nt), C.byref(cv))
            N.call("mglp_engine_backward_keep_grads", self.h, cfg["B"], cfg["sx"], cfg["sy"],
                   None, N.dptr(self.lamh), N.dptr(lam0), N.dptr(tr), 64, C.byref(nt),
                   C.byref(cv))
        one()
        if self.dist is not None:
            self.dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k):
            one()
        torch.cuda.synchronize()
        ms = self.max_over_ranks((time.perf_counter() - t0) * 1e3 / k)
        sb = 4 * self.n_state
        return {"value": ms, "unit": "ms/iteration", "h2d_bytes_per_step": 2 * sb,
                "d2h_bytes_per_step": sb + 2 * 64 * 8,
                "api": "mglp_engine_forward + mglp_engine_backward_keep_grads (host f64 z0, "
                       "lambda_N -> lambda_0, traces; gradients stay in the device slab)"}

    def e2e_host_grads(self, k):
        """the reference's exact call shape: trajectory AND every parameter
        gradient accumulated into caller-owned host f64 arrays each step
        (mglp_engine_forward traj_out + mglp_engine_backward grads_accum)"""
        N, np, torch = self.N, self.np, self.torch
        cfg = self.cfg
        total = cfg["n_enc"] + cfg["n_dec"]
        npar = C.c_longlong()
        N.call("mglp_engine_info", self.h, None, None, None, C.byref(npar))
        grads = np.zeros(npar.value)
        traj = np.empty((total + 1) * self.n_logical)
        lam0 = np.empty(self.n_logical)
        tr = np.empty(64)
        nt, cv = C.c_int(), C.c_int()

        def one():
            N.call("mglp_engine_forward", self.h, cfg["B"], cfg["sx"], cfg["sy"],
                   N.dptr(self.z0h), N.dptr(traj), N.dptr(tr), 64, C.byref(nt), C.byref(cv))
            N.call("mglp_engine_backward", self.h, cfg["B"], cfg["sx"], cfg["sy"], None,
                   N.dptr(self.lamh), N.dptr(lam0), N.dptr(grads), N.dptr(tr), 64,
                   C.byref(nt), C.byref(cv))
        one()
        t0 = time.perf_counter()
        for _ in range(k):
            one()
        ms = (time.perf_counter() - t0) * 1e3 / k
        return {"value": ms, "unit": "ms/iteration", "steps": k,
                "h2d_bytes_per_step": 2 * 4 * self.n_state,
                "d2h_bytes_per_step": 4 * (self.n_state * (total + 2) + npar.value),
                "api": "mglp_engine_forward(traj_out) + mglp_engine_backward(grads_accum): "
                       f"{total + 1} host f64 states + {npar.value} host f64 gradients per step"}


def trainer_e2e(cfg, local, k):
    """mglp_trainer_update (training.cpp:202-268 run_update on the device:
    make_batch, embedding, the engine solve, head + cross entropy, adjoint,
    embedding backward, AdamW) on the config's stack, copy_sequence task,
    vocab 1024; wall clock per update with the loss read back."""
    from paper_2601_09026_b200 import _native as N
    from paper_2601_09026_b200.engine import SolveConfig, StackConfig
    sc = StackConfig(kind=cfg["kind"], d=cfg["d"], heads=cfg["H"], ffn=cfg["ffn"],
                     n_enc=cfg["n_enc"], n_dec=cfg["n_dec"])
    so = SolveConfig(coarsen=cfg["cf"], levels=cfg["levels"], fwd_iters=cfg["fwd"],
                     bwd_iters=cfg["bwd"], warm_start=False)
    kind = {"encoder": 0, "decoder_only": 0, "encoder_decoder": 2}[cfg["kind"]]
    task = N.TaskDesc(kind, 1024, cfg["sx"], cfg["B"] * 64, cfg["B"], 1)
    opt = N.OptDesc(2, 1e-3, 0.9, 0.999, 1e-8, 0.01, 0.0)
    h = C.c_void_p()
    N.call("mglp_trainer_create", C.byref(sc.desc()), C.byref(so.desc()), C.byref(task),
           C.byref(opt), 1024, cfg["sx"], cfg["B"], 7, local, C.byref(h))
    try:
        loss = C.c_double()
        for i in range(3):
            N.call("mglp_trainer_update", h, i, 1, 1, C.byref(loss))
        t0 = time.perf_counter()
        for i in range(k):
            N.call("mglp_trainer_update", h, 3 + i, 1, 1, C.byref(loss))
        ms = (time.perf_counter() - t0) * 1e3 / k
    finally:
        N.call("mglp_trainer_destroy", h)
    return {"value": ms, "unit": "ms/update", "steps": k, "loss_last": loss.value,
            "api": "mglp_trainer_update (device make_batch + embed + engine fwd/bwd + head/CE + "
                   "embed backward + AdamW; loss to host)", "task": "copy_sequence vocab 1024"}


def serial_reference_ms(name, args, local):
    """device serial fwd+bwd (serial_forward + serial_adjoint with gradients,
    activation caching) of the FULL stack on ONE GPU: the speedup baseline"""
    r = DeviceRun(name, args, 0, 1, None, local)
    try:
        for _ in range(max(2, args.warmup // 2)):
            r.serial_step()
        return r.device_timed(r.serial_step, max(2, min(args.steps // 2, 10)))
    finally:
        r.close()


def measure(name, args, rank, world, dist, local, headline):
    """One config: timed MGRIT iterations, serial baseline, probe step,
    profile (roofline), e2e. Returns the result dict on rank 0."""
    cfg = CONFIGS[name]
    steps = args.steps if headline else max(3, min(args.steps, args.extra_steps))
    r = DeviceRun(name, args, rank, world, dist, local)
    res = {}
    try:
        for _ in range(args.warmup):
            r.eager_step()
        r.N.call("mglp_engine_sync", r.h)
        note = None if args.no_graph else r.capture()
        r.launches()
        with ClockSampler(local) as clk:
            ms = r.device_timed(r.step, steps)
        launches = r.launches()
        fwd_trace, bwd_trace = r.traces()
        backend, nranks = r.comm_info()
        probe_ms, probe_note = r.probe_ms() if (headline or cfg["levels"] > 2) else (None, None)
        ms3, fl3, by3, ln3 = r.profile()
        e2e = r.e2e(steps)
        e2e_host = r.e2e_host_grads(2) if (headline and world == 1 and args.host_grads) else None
        res = {"ms": ms, "steps": steps, "launches": launches, "fwd_trace": fwd_trace,
               "bwd_trace": bwd_trace, "probe_ms": probe_ms, "probe_note": probe_note,
               "prof": (ms3, fl3, by3, ln3), "e2e": e2e, "e2e_host": e2e_host,
               "clocks": clk.summary(), "graph_note": note, "backend": backend,
               "backend_nranks": nranks}
    finally:
        r.close()
    # serial baseline of the full stack on one GPU (rank 0; the others wait)
    serial = None
    if rank == 0:
        serial = serial_reference_ms(name, args, local)
    if dist is not None:
        dist.barrier()
    if rank != 0:
        return None
    res["serial_ms"] = serial
    return res


def summarize(name, res, world, peaks):
    cfg = CONFIGS[name]
    ms3, fl3, by3, ln3 = res["prof"]
    bf16 = peaks.get("bf16_tflops_sustained", 1400.0)
    gemm_ms, gemm_fl = ms3[0], fl3[0]
    achieved = gemm_fl / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else 0.0
    out = {
        "ms_per_iteration": res["ms"], "steps": res["steps"],
        "serial_ms_per_step": res["serial_ms"],
        "speedup_vs_serial": res["serial_ms"] / res["ms"] if res["serial_ms"] else None,
        "fwd_trace": res["fwd_trace"], "bwd_trace": res["bwd_trace"],
        "gemm_tflops": achieved, "gemm_frac_of_bf16": achieved / bf16,
        "gemm_frac_of_split_ceiling": achieved / (bf16 / 3.0),
        "attention_tflops": fl3[1] / (ms3[1] * 1e-3) / 1e12 if ms3[1] > 0 else None,
        "per_class_ms_rank0": {"gemm_tcgen05": ms3[0], "attention_tcgen05": ms3[1],
                               "rows_layernorm_colsum_state": ms3[2]},
        "e2e": res["e2e"], "gpu_launches": res["launches"], "clocks": res["clocks"],
        "comm": {"backend": res["backend"], "nranks_reported": res["backend_nranks"]},
    }
    if res["probe_ms"] is not None:
        out["monitor_probe_ms_per_step"] = res["probe_ms"]
        out["monitor_probe_budget"] = res["probe_note"]
    return out


def run_device(args, rank, world, dist):
    import torch
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    head = measure(args.config, args, rank, world, dist, local, headline=True)
    extras = {}
    if not args.no_extra:
        from paper_2601_09026_b200 import dist as D
        for name in [x for x in args.extra.split(",") if x and x != args.config]:
            c = CONFIGS[name]
            try:
                D.check_partition(c["n_enc"] + c["n_dec"], c["cf"], c["levels"], world)
            except Exception as ex:  # noqa: BLE001
                extras[name] = {"skipped": str(ex)}
                continue
            r = measure(name, args, rank, world, dist, local, headline=False)
            if rank == 0:
                extras[name] = summarize(name, r, world, peaks)
    trainer = None
    if rank == 0 and world == 1 and not args.no_trainer:
        try:
            trainer = trainer_e2e(CONFIGS[args.config], local, max(3, min(args.steps, 10)))
        except Exception as ex:  # noqa: BLE001 -- reported, never fatal
            trainer = {"error": str(ex)}
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    s = summarize(args.config, head, world, peaks)
    ms3, fl3, by3, ln3 = head["prof"]
    bf16 = peaks.get("bf16_tflops_sustained", 1400.0)
    traffic, traffic_src = traffic_evidence()
    roofline = {
        "kernel": "gemm_tc_kernel (tcgen05 kind::f16, 3-pass fp16 hi/lo split, fp32 accumulate)",
        "bound": "tensor", "achieved": s["gemm_tflops"], "peak": bf16, "unit": "TFLOP/s",
        "frac": s["gemm_tflops"] / bf16,
        "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (measured)",
        "traffic": traffic, "traffic_unit": "bytes per launch (dram read + write)",
        "traffic_source": traffic_src,
        "achieved_how": "algorithmic GEMM FLOPs of one profiled iteration (rank 0) / sum of "
                        "CUDA-event durations of its GEMM launches (engine stream)",
        "frac_of_split_ceiling": s["gemm_frac_of_split_ceiling"],
        "gemm_share_of_step": ms3[0] / sum(ms3) if sum(ms3) > 0 else None,
        "gemm_launches_per_step": ln3[0],
        "attention": {"achieved": s["attention_tflops"], "unit": "TFLOP/s",
                      "launches_per_step": ln3[1]},
        "per_class_ms": s["per_class_ms_rank0"],
    }
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref as R
            if R.available():
                threads = max(1, min(os.cpu_count() or 1, cfg["n_enc"] + cfg["n_dec"]))
                smp = reference_sample(cfg, threads)
                cpu = {"value": smp["ms"], "unit": "ms/iteration", "cores": threads,
                       "kind": "reference", "sample": smp["sample"],
                       "serial_ms": smp["serial_ms"]}
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "error": str(ex)}
    line = {
        "metric": METRIC, "value": head["ms"], "unit": "ms/iteration", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms"],
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (reference LayerStack init seed 7; z0/lambda_N from rng::gaussian)",
        "config": dict(config_block(args.config, cfg, world),
                       launch="CUDA graph of the whole step" if not head["graph_note"] and
                       not args.no_graph else (head["graph_note"] or "eager")),
        "speedup_vs_serial": s["speedup_vs_serial"],
        "serial_ms_per_step": s["serial_ms_per_step"],
        "monitor_probe_ms_per_step": s.get("monitor_probe_ms_per_step"),
        "monitor_probe_budget": s.get("monitor_probe_budget"),
        "fwd_trace": s["fwd_trace"], "bwd_trace": s["bwd_trace"],
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": head["e2e"],
        "e2e_host_grads": head["e2e_host"],
        "e2e_trainer_update": trainer,
        "comm": s["comm"],
        "gpu_launches": head["launches"],
        "clocks": head["clocks"],
        "configs": extras,
    }
    print(json.dumps(line), flush=True)


def dry_run(args, rank, world):
    """The launch path without a GPU: world ranks over gloo, each reporting
    the layer block it would own for every config (dist.owned_layers, the
    engine's partition); rank 0 prints one JSON line."""
    from paper_2601_09026_b200 import dist as D
    blocks = {}
    for name, c in CONFIGS.items():
        n = c["n_enc"] + c["n_dec"]
        try:
            blocks[name] = list(D.owned_layers(n, c["cf"], c["levels"], rank, world))
        except Exception as ex:  # noqa: BLE001
            blocks[name] = str(ex)
    got = [blocks]
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        got = [None] * world
        dist.all_gather_object(got, blocks)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world,
                          "gpus_arg": args.gpus, "ranks": got}), flush=True)
    return 0


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn(args):
    """--gpus N without a launcher: re-run this script under torchrun with N
    ranks (one process per GPU); rank 0's JSON line is the output."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and not args.dry_run:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but only {have} "
                                                     f"CUDA devices visible"}))
        return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="bert", choices=sorted(CONFIGS))
    ap.add_argument("--extra", default="tiny,gpt,vit,mt",
                    help="further BASELINE configs timed in the same run (line['configs'])")
    ap.add_argument("--extra-steps", type=int, default=5)
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-trainer", action="store_true")
    ap.add_argument("--host-grads", type=int, default=1,
                    help="also time the host-f64-gradient call shape (headline, N=1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels eagerly")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: spawn/rendezvous over gloo and print each rank's layer block "
                         "(the CPU test of the --gpus N launch path)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    return args


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    world = int(env_world or "1")
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, CONFIGS[args.config], rank, world)
        return 0
    if env_world is None and args.gpus > 1:
        return spawn(args)
    if world != args.gpus:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "error": f"WORLD_SIZE={world} but --gpus "
                                                         f"{args.gpus}"}))
        return 1
    if args.dry_run:
        return dry_run(args, rank, world)
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist  # noqa: F811
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        # NCCL's own record of the communicators (ranks, NVLink/NVLS paths)
        logdir = os.path.join(ROOT, "gpurun_out", "nccl")
        os.makedirs(logdir, exist_ok=True)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(logdir, f"nccl.rank{rank}.%p.log"))
        dist.init_process_group("nccl")
    run_device(args, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
