"""ctypes binding of libparnn_b200.so (include/parnn_b200.h).

The library is built in-tree by ``make -C paper_1507_01239_b200`` (see
``__graft_entry__.build``). There is no fallback: if the library is missing
every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libparnn_b200.so")

c_u64 = C.c_uint64
c_f64 = C.c_double
c_int = C.c_int
vp = C.c_void_p


class ParnnError(RuntimeError):
    """Mirror of parnn::Error (error.hpp:12-15): the message names the op and values."""


class TrainConfig(C.Structure):
    """parnn_train_config (include/parnn_b200.h)."""
    _fields_ = [("workers", c_u64), ("avg_frequency", c_u64), ("minibatch", c_u64), ("base_seed", c_u64),
                ("optimizer", c_int), ("lr_schedule", c_int), ("lr_init", c_f64), ("epochs", c_u64),
                ("ng_decay", c_f64), ("ng_smoothing", c_f64), ("precision", c_int), ("activation", c_int),
                ("rank0", c_u64), ("local_workers", c_u64), ("serial", c_int),
                ("ng_rank_in", c_int), ("ng_rank_out", c_int), ("ng_update_period", c_int), ("ng_history", c_f64),
                ("ng_update_lag", c_int)]


# (name, restype, argtypes) for every symbol declared in include/parnn_b200.h
SIGNATURES = [
    ("parnn_last_error", C.c_char_p, []),
    ("parnn_version", C.c_char_p, []),
    ("parnn_rng_u64", c_int, [c_u64, c_u64, vp]),
    ("parnn_rng_uniform", c_int, [c_u64, c_u64, vp]),
    ("parnn_rng_gaussian", c_int, [c_u64, c_u64, c_f64, c_f64, vp]),
    ("parnn_shuffled_indices", c_int, [c_u64, c_u64, vp]),
    ("parnn_partition_rows", c_int, [c_u64, c_u64, c_u64, vp]),
    ("parnn_minibatch_rows", c_int, [c_u64, c_u64, c_u64, vp]),
    ("parnn_make_data", c_int, [c_u64, c_u64, c_u64, c_f64, c_u64, c_f64, c_u64, c_int, vp, vp, vp, vp, vp, vp]),
    ("parnn_param_count", c_u64, [vp, c_int]),
    ("parnn_init_random", c_int, [vp, c_int, c_u64, vp]),
    ("parnn_exponential_lr", c_int, [c_f64, c_u64, c_f64, vp]),
    ("parnn_newbob_sequence", c_int, [c_f64, vp, c_u64, vp, vp]),
    ("parnn_scale_lr_for_workers", c_int, [c_f64, c_u64, vp]),
    ("parnn_save_model", c_int, [C.c_char_p, vp, c_int, c_int, vp]),
    ("parnn_load_model", c_int, [C.c_char_p, vp, vp, vp, vp, c_u64]),
    ("parnn_lowrank_basis", c_int, [c_u64, c_u64, c_u64, vp]),
    ("parnn_debug_lowrank_eig", c_int, [c_int, c_u64, c_f64, c_f64, c_f64, vp, vp, vp, vp, vp]),
    ("parnn_lowrank_seed", c_u64, [c_int, c_int]),
    ("parnn_debug_gemm", c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                 c_int, c_int, C.c_float, C.c_float, C.c_float, vp, vp, vp, vp, vp, vp, vp, vp]),
    ("parnn_allreduce_average_host", c_int, [vp, c_u64, c_u64, vp]),
    ("parnn_ctx_create", c_int, [c_int, vp]),
    ("parnn_ctx_destroy", c_int, [vp]),
    ("parnn_ctx_sync", c_int, [vp]),
    ("parnn_dataset_create", c_int, [vp, vp, vp, c_u64, c_u64, c_u64, vp]),
    ("parnn_dataset_destroy", c_int, [vp]),
    ("parnn_dataset_generate", c_int, [vp, c_u64, c_u64, c_u64, c_f64, c_u64, c_f64, c_u64, c_int, vp, vp]),
    ("parnn_dataset_info", c_int, [vp, vp, vp, vp]),
    ("parnn_dataset_download", c_int, [vp, vp, vp]),
    ("parnn_load_csv", c_int, [C.c_char_p, vp, vp, c_u64, c_u64, vp, vp, vp]),
    ("parnn_dataset_load_csv", c_int, [vp, C.c_char_p, vp]),
    ("parnn_save_csv", c_int, [C.c_char_p, vp, vp, c_u64, c_u64]),
    ("parnn_replica_create", c_int, [vp, vp, c_int, c_int, c_int, c_int, c_u64, c_u64, c_f64, c_f64, vp]),
    ("parnn_replica_destroy", c_int, [vp]),
    ("parnn_replica_set_params", c_int, [vp, vp, c_u64]),
    ("parnn_replica_get_params", c_int, [vp, vp, c_u64]),
    ("parnn_replica_get_ng_state", c_int, [vp, vp, c_u64]),
    ("parnn_replica_set_ng_state", c_int, [vp, vp, c_u64, c_u64]),
    ("parnn_replica_set_lowrank", c_int, [vp, c_int, c_int, c_int, c_int, c_f64, c_int]),
    ("parnn_replica_lowrank_state", c_int, [vp, c_int, c_int, vp, vp, vp, vp, vp]),
    ("parnn_replica_lowrank_diag", c_int, [vp, c_int, c_int, vp]),
    ("parnn_replica_bind", c_int, [vp, vp]),
    ("parnn_replica_upload_epoch", c_int, [vp, vp, vp, c_u64]),
    ("parnn_replica_step", c_int, [vp, c_u64]),
    ("parnn_replica_sync", c_int, [vp]),
    ("parnn_replica_ce", c_int, [vp, vp, c_u64]),
    ("parnn_replica_step_ce", c_int, [vp, c_u64, vp]),
    ("parnn_replica_forward", c_int, [vp, vp, vp, c_u64, vp]),
    ("parnn_replica_accuracy", c_int, [vp, vp, vp]),
    ("parnn_replica_kernels_per_step", c_int, [vp, vp]),
    ("parnn_replica_time_steps", c_int, [vp, c_u64, vp]),
    ("parnn_replica_profile", c_int, [vp, c_u64, vp, c_u64, vp, vp, c_u64, vp]),
    ("parnn_dataset_write_f32", c_int, [vp, vp, vp, c_u64, c_u64]),
    ("parnn_comm_unique_id", c_int, [vp]),
    ("parnn_comm_create", c_int, [vp, vp, c_int, c_int, vp]),
    ("parnn_comm_destroy", c_int, [vp]),
    ("parnn_average", c_int, [vp, c_int, vp, c_u64]),
    ("parnn_run_steps", c_int, [vp, c_int, vp, c_u64, c_u64, c_u64, vp]),
    ("parnn_time_average", c_int, [vp, c_int, vp, c_u64, c_u64, vp, vp]),
    ("parnn_averager_create", c_int, [vp, c_int, vp, c_u64, vp]),
    ("parnn_averager_run", c_int, [vp]),
    ("parnn_averager_destroy", c_int, [vp]),
    ("parnn_train", c_int, [vp, vp, vp, vp, c_int, vp, vp, vp, vp, vp, vp]),
    ("parnn_rbm_create", c_int, [vp, c_u64, c_u64, c_int, c_u64, c_int, vp]),
    ("parnn_rbm_destroy", c_int, [vp]),
    ("parnn_rbm_set_params", c_int, [vp, vp]),
    ("parnn_rbm_get_params", c_int, [vp, vp]),
    ("parnn_rbm_cd1", c_int, [vp, vp, c_u64, c_f64, c_int, c_u64, c_u64, vp]),
    ("parnn_rbm_hidden_probs", c_int, [vp, vp, c_u64, vp]),
    ("parnn_rbm_reconstruction_error", c_int, [vp, vp, c_u64, vp]),
    ("parnn_greedy_pretrain", c_int, [vp, vp, c_int, vp, c_u64, c_u64, c_f64, c_f64, c_u64, c_u64, c_int, vp]),
    ("parnn_greedy_pretrain_rng", c_int, [vp, vp, c_int, vp, c_u64, c_u64, c_f64, c_f64, c_u64, c_int, vp, vp, vp,
                                          c_int, vp]),
    ("parnn_pretrain_last_stats", c_int, [vp, vp, vp]),
]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ParnnError(f"{LIB_PATH} is missing: build it with `make -C {HERE}` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise ParnnError(lib().parnn_last_error().decode())


def ptr(a: np.ndarray):
    return a.ctypes.data_as(vp)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)
