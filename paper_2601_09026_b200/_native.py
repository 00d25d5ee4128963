"""ctypes binding of the C-ABI in include/mglp_cuda.h (libmglp_cuda.so).

There is no fallback: if the in-tree CUDA library is missing, or no GPU is
visible when a device call is made, the call raises. The product path never
touches oracle/.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libmglp_cuda.so")


class ValidationError(ValueError):
    """Bad input or configuration (reference errors.hpp:25-29, status 1)."""


class ContractViolation(RuntimeError):
    """Broken internal invariant or CUDA failure (errors.hpp:31-35, status 2)."""


class StackDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("d", C.c_int), ("heads", C.c_int), ("ffn", C.c_int),
                ("n_enc", C.c_int), ("n_dec", C.c_int), ("buffer_open", C.c_int),
                ("buffer_close", C.c_int), ("ln_eps", C.c_double), ("base_h", C.c_double),
                ("dropout", C.c_double), ("init_std", C.c_double),
                ("depth_scaled_init", C.c_int)]


class TaskDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("vocab", C.c_int), ("seq_len", C.c_int),
                ("train_size", C.c_int), ("val_size", C.c_int), ("seed", C.c_ulonglong)]


class OptDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("lr", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("weight_decay", C.c_double),
                ("momentum", C.c_double)]


class SolveDesc(C.Structure):
    _fields_ = [("coarsen", C.c_int), ("levels", C.c_int), ("fwd_iters", C.c_int),
                ("bwd_iters", C.c_int), ("fwd_tol", C.c_double), ("bwd_tol", C.c_double),
                ("cold_guess", C.c_int), ("warm_start", C.c_int)]


_lib = None
_loaded_path = None

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)
_llp = C.POINTER(C.c_longlong)
_vp = C.c_void_p

_SIGS = {
    "mglp_engine_create": [C.POINTER(StackDesc), C.POINTER(SolveDesc), C.c_int, C.POINTER(_vp)],
    "mglp_engine_destroy": [_vp],
    "mglp_engine_info": [_vp, _ip, _ip, _ip, _llp],
    "mglp_engine_step_size": [_vp, C.c_int, _dp],
    "mglp_engine_init_params": [_vp, C.c_ulonglong, _dp],
    "mglp_engine_set_params": [_vp, _dp, C.c_longlong],
    "mglp_engine_get_params": [_vp, _dp, C.c_longlong],
    "mglp_engine_get_config": [_vp, C.POINTER(SolveDesc)],
    "mglp_engine_set_config": [_vp, C.POINTER(SolveDesc)],
    "mglp_engine_forward": [_vp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, C.c_int, _ip, _ip],
    "mglp_engine_backward": [_vp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_int,
                             _ip, _ip],
    "mglp_engine_backward_keep_grads": [_vp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp,
                                        C.c_int, _ip, _ip],
    "mglp_engine_comm_info": [_vp, _ip, _ip],
    "mglp_engine_memory": [_vp, _llp],
    "mglp_engine_set_dropout_masks": [_vp, C.c_int, C.c_int, C.c_int, _vp],
    "mglp_engine_snapshot": [_vp],
    "mglp_engine_restore": [_vp],
    "mglp_engine_snapshot_id": [_vp, C.POINTER(C.c_longlong)],
    "mglp_engine_restore_id": [_vp, C.c_longlong],
    "mglp_engine_seed_forward_from_traj": [_vp],
    "mglp_engine_reset": [_vp],
    "mglp_serial_forward": [_vp, C.c_int, C.c_int, C.c_int, _dp, _dp],
    "mglp_serial_adjoint": [_vp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp],
    "mglp_stack_step": [_vp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, _dp, _dp],
    "mglp_stack_adjoint_step": [_vp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, _dp, _dp,
                                _dp, C.c_double, _dp],
    "mglp_engine_set_shape": [_vp, C.c_int, C.c_int, C.c_int, _llp],
    "mglp_engine_stream": [_vp, C.POINTER(_vp)],
    "mglp_engine_forward_device": [_vp, _vp],
    "mglp_engine_backward_device": [_vp, _vp, _vp, C.c_int],
    "mglp_serial_forward_device": [_vp, _vp],
    "mglp_serial_adjoint_device": [_vp, _vp, _vp, C.c_int],
    "mglp_engine_zero_grads": [_vp],
    "mglp_engine_graph_capture": [_vp, _vp, _vp, _vp, C.c_int],
    "mglp_engine_graph_replay": [_vp],
    "mglp_engine_get_grads": [_vp, _dp, C.c_longlong],
    "mglp_engine_get_grads_layers": [_vp, C.c_int, C.c_int, _dp, C.c_longlong],
    "mglp_engine_read_traj": [_vp, C.c_int, C.c_int, _vp],
    "mglp_engine_trace": [_vp, C.c_int, _dp, C.c_int, _ip, _ip],
    "mglp_engine_traj_device": [_vp, C.POINTER(_vp)],
    "mglp_engine_sync": [_vp],
    "mglp_engine_take_launch_count": [_vp, _llp],
    "mglp_monitor_record": [_vp, C.c_longlong, _ip],
    "mglp_engine_monitor_attach": [_vp, C.c_double, C.c_int, C.c_int],
    "mglp_engine_monitor_probe": [_vp, C.c_int],
    "mglp_engine_monitor_read": [_vp, _ip, _ip, _dp, _dp, _ip, _ip, _ip, _ip],
    "mglp_engine_monitor_reports": [_vp, _llp, _dp, _dp, _ip, C.c_int, _ip],
    "mglp_engine_capture_cycles": [_vp, C.c_int],
    "mglp_trainer_monitor_attach": [_vp, C.c_double, C.c_int, C.c_int],
    "mglp_trainer_update_probe": [_vp, C.c_longlong, C.c_int, _dp, _ip, _ip, _dp, _dp, _ip, _ip],
    "mglp_trainer_last_factors": [_vp, _dp, _dp, _ip, _ip],
    "mglp_trainer_monitor_reports": [_vp, _llp, _dp, _dp, _ip, C.c_int, _ip],
    "mglp_engine_profile": [_vp, C.c_int],
    "mglp_rng_gaussian_fill": [C.c_ulonglong, C.c_ulonglong, C.c_ulonglong, C.c_double, _dp,
                               C.c_longlong],
    "mglp_engine_profile_read": [_vp, _dp, _dp, _dp, _llp],
    "mglp_engine_profile_dump": [_vp, _dp, C.c_int, _ip],
    "mglp_nccl_unique_id": [_vp],
    "mglp_engine_create_dist": [C.POINTER(StackDesc), C.POINTER(SolveDesc), C.c_int, C.c_int,
                                C.c_int, _vp, C.POINTER(_vp)],
    "mglp_engine_rank_info": [_vp, _ip, _ip, _ip, _ip],
    "mglp_loopback_create": [C.POINTER(StackDesc), C.POINTER(SolveDesc), C.c_int, C.c_int,
                             C.POINTER(_vp)],
    "mglp_loopback_run_fwd_bwd": [C.POINTER(_vp), C.c_int, _vp, _vp, _vp, C.c_int],
    "mglp_test_gemm": [C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.c_longlong, C.c_int, C.c_int,
                       _vp, C.c_longlong, C.c_int, C.c_int, C.c_int, _vp, _vp, C.c_longlong,
                       C.c_int, C.c_int, _ip],
    "mglp_trainer_create": [C.POINTER(StackDesc), C.POINTER(SolveDesc), C.POINTER(TaskDesc),
                            C.POINTER(OptDesc), C.c_int, C.c_int, C.c_int, C.c_ulonglong,
                            C.c_int, C.POINTER(_vp)],
    "mglp_trainer_destroy": [_vp],
    "mglp_trainer_update": [_vp, C.c_longlong, C.c_int, C.c_int, _dp],
    "mglp_trainer_evaluate": [_vp, _dp],
    "mglp_trainer_num_params": [_vp, _llp],
    "mglp_trainer_get_params": [_vp, _dp],
    "mglp_trainer_set_params": [_vp, _dp],
    "mglp_trainer_get_grads": [_vp, _dp],
    "mglp_trainer_read_logits": [_vp, _fp],
    "mglp_trainer_read_batch": [_vp, C.c_int, C.c_longlong, _ip, _ip, _ip],
    "mglp_trainer_get_iters": [_vp, _ip, _ip],
    "mglp_trainer_set_iters": [_vp, C.c_int, C.c_int],
    "mglp_trainer_snapshot": [_vp],
    "mglp_trainer_restore": [_vp],
    "mglp_trainer_trace": [_vp, C.c_int, _dp, C.c_int, _ip, _ip],
    "mglp_trainer_save_checkpoint": [_vp, C.c_longlong, C.c_char_p, C.c_longlong, C.c_char_p,
                                     C.c_longlong, _llp],
    "mglp_trainer_load_checkpoint": [_vp, C.c_char_p, C.c_longlong, _llp, C.c_char_p,
                                     C.c_longlong, _llp, _ip],
    "mglp_bench_gemm": [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                        C.c_int, C.POINTER(C.c_float)],
    "mglp_test_attention": [C.c_int] * 6 + [_vp, _vp, _vp, C.c_int] + [_vp] * 6 + [_ip],
    "mglp_bench_attention": [C.c_int] * 8 + [C.POINTER(C.c_float)],
    "mglp_engine_refresh_dropout": [_vp, C.c_ulonglong, C.c_ulonglong, C.c_int, C.c_int, C.c_int],
    "mglp_engine_clear_dropout": [_vp],
    "mglp_engine_lipschitz": [_vp, C.c_int, C.c_double, C.c_double, C.c_int, C.c_ulonglong, _ip,
                              C.c_int, _dp],
}

EXPORTS = sorted(list(_SIGS) + ["mglp_last_error", "mglp_version"])


def lib_path() -> str:
    return os.environ.get("MGLP_LIB", LIB_PATH)


def lib():
    """Load the in-tree CUDA library (raises if it was never built)."""
    global _lib, _loaded_path
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise RuntimeError(
            f"mglp CUDA library not found at {path}: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (make -C "
            "paper_2601_09026_b200/csrc). There is no CPU fallback.")
    L = C.CDLL(path)
    L.mglp_last_error.restype = C.c_char_p
    L.mglp_version.restype = C.c_char_p
    for name, args in _SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    _lib, _loaded_path = L, path
    return L


def check(status: int):
    if status == 0:
        return
    msg = lib().mglp_last_error().decode()
    if status == 1:
        raise ValidationError(msg)
    raise ContractViolation(msg)


def call(name, *args):
    check(getattr(lib(), name)(*args))


def dptr(a):
    """float64 numpy array -> double* (None -> NULL)."""
    if a is None:
        return None
    return a.ctypes.data_as(_dp)
