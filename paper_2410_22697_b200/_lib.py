"""ctypes binding of libmgnn.so (include/mgnn.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MGNN_LIB", os.path.join(HERE, "libmgnn.so"))   # override: A/B builds

MAX_LAYERS = 8
PROF_N = 16                      # MGNN_PROF_N
IPC_HANDLE_BYTES = 64
C_NODES, C_LOCAL, C_HIT, C_MISS, C_EVICTED, C_REFILLED, C_ROWS_FETCHED, C_PEER_ROWS, C_N = 0, 1, 2, 3, 4, 5, 6, 7, 8
STATUS = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 5: "ESTATE", 6: "EOVERFLOW"}

# every symbol include/mgnn.h declares (checked by tests/test_abi.py)
SYMBOLS = [
    "mgnn_alpha_default", "mgnn_ctx_create", "mgnn_destroy", "mgnn_last_error", "mgnn_partition_load",
    "mgnn_table_export", "mgnn_table_import", "mgnn_buffer_init", "mgnn_sampler_config", "mgnn_sample",
    "mgnn_lookup_gather", "mgnn_score_evict_refill", "mgnn_sampler_config_bounded", "mgnn_window_get", "mgnn_counts_read",
    "mgnn_counts_read_async",
    "mgnn_buffer_snapshot", "mgnn_part_info", "mgnn_next_step", "mgnn_window_shape", "mgnn_window_bind_x",
    "mgnn_sampler_defer_relabel", "mgnn_relabel", "mgnn_halo_get", "mgnn_table_row", "mgnn_launch_count",
    "mgnn_profile_enable", "mgnn_profile_read", "mgnn_profile_stages", "mgnn_profile_kernels",
    "mgnn_sage_config", "mgnn_sage_forward", "mgnn_sage_train_config", "mgnn_sage_train_step",
    "mgnn_sage_grads", "mgnn_sage_sgd", "mgnn_sage_loss", "mgnn_sage_params", "mgnn_sampler_expand_remote",
    "mgnn_graph_csr_load", "mgnn_ctx_set_dense_scores", "mgnn_sm_partition",
]


class PartitionDesc(C.Structure):
    _fields_ = [("part_id", C.c_int32), ("indptr", C.c_void_p), ("cols", C.c_void_p),
                ("train_ids", C.c_void_p), ("n_train", C.c_int64)]


class Policy(C.Structure):
    _fields_ = [("gamma", C.c_float), ("alpha", C.c_float), ("theta_r", C.c_float),
                ("delta", C.c_int32), ("f_bp", C.c_uint32)]


class Window(C.Structure):
    _fields_ = [("n_inst", C.c_int32), ("n_steps", C.c_int32), ("n_parts_local", C.c_int32),
                ("n_layers", C.c_int32), ("step0", C.c_uint64), ("rows_stride", C.c_int64),
                ("pitch", C.c_int64), ("X", C.c_void_p), ("frontier", C.c_void_p), ("hop_size", C.c_void_p),
                ("offsets", C.c_void_p * MAX_LAYERS), ("cols", C.c_void_p * MAX_LAYERS),
                ("off_stride", C.c_int64 * MAX_LAYERS), ("col_stride", C.c_int64 * MAX_LAYERS),
                ("counts", C.c_void_p)]


class SageDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("dims", C.c_void_p), ("w_self", C.c_void_p),
                ("w_neigh", C.c_void_p), ("bias", C.c_void_p)]


class MgnnError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn}: {STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load(path: str = LIB_PATH):
    """Load libmgnn.so; raises if it is missing (no fallback of any kind)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libmgnn.so not built at {path}: run python -m paper_2410_22697_b200.build")
    L = C.CDLL(path)
    P, I32, I64, U32, U64, F32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float
    S = C.c_int
    sig = {
        "mgnn_alpha_default": (F32, [F32, I32]),
        "mgnn_ctx_create": (S, [I32, I32, I64, P, I32, U64, P]),
        "mgnn_destroy": (None, [P]),
        "mgnn_last_error": (C.c_char_p, [P]),
        "mgnn_partition_load": (S, [P, P, P]),
        "mgnn_table_export": (S, [P, I32, P]),
        "mgnn_table_import": (S, [P, I32, P]),
        "mgnn_buffer_init": (S, [P, P, P]),
        "mgnn_sampler_config": (S, [P, P, I32, I32, U64, I32]),
        "mgnn_sampler_config_bounded": (S, [P, P, I32, I32, U64, I32, I64]),
        "mgnn_sample": (S, [P, I32, U64, I32, P, P, I32, P]),
        "mgnn_lookup_gather": (S, [P, I32, P]),
        "mgnn_score_evict_refill": (S, [P, I32, P]),
        "mgnn_window_get": (S, [P, I32, P]),
        "mgnn_counts_read": (S, [P, I32, P, P]),
        "mgnn_counts_read_async": (S, [P, I32, P, P]),
        "mgnn_buffer_snapshot": (S, [P, I32, P, P, P, P, P]),
        "mgnn_part_info": (S, [P, I32, P]),
        "mgnn_halo_get": (S, [P, I32, P, P]),
        "mgnn_table_row": (S, [P, I64, P]),
        "mgnn_launch_count": (I64, [P]),
        "mgnn_next_step": (S, [P, P]),
        "mgnn_window_shape": (S, [P, P, P, P]),
        "mgnn_sampler_defer_relabel": (S, [P, I32]),
        "mgnn_relabel": (S, [P, I32, P]),
        "mgnn_sm_partition": (S, [P, I32, P]),
        "mgnn_window_bind_x": (S, [P, I32, P, I64]),
        "mgnn_profile_enable": (S, [P, I32]),
        "mgnn_profile_read": (S, [P, P, P, P]),
        "mgnn_profile_stages": (S, [P, P, I32]),
        "mgnn_profile_kernels": (S, [I32, P, I64]),
        "mgnn_sage_config": (S, [P, P]),
        "mgnn_sage_forward": (S, [P, I32, P, I64, P]),
        "mgnn_sage_train_config": (S, [P, P]),
        "mgnn_sage_train_step": (S, [P, I32, I32, I32, P]),
        "mgnn_sage_grads": (S, [P, P, P]),
        "mgnn_sage_sgd": (S, [P, F32, P]),
        "mgnn_sage_loss": (S, [P, P, P]),
        "mgnn_sage_params": (S, [P, I32, P, P, P]),
        "mgnn_sampler_expand_remote": (S, [P, I32]),
        "mgnn_graph_csr_load": (S, [P, P, P]),
        "mgnn_ctx_set_dense_scores": (S, [P, I32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L
