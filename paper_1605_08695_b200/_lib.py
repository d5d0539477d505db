"""ctypes binding of libtfs.so (include/tfs.h).  Argument marshalling only.

The shared library is built in-tree by ``paper_1605_08695_b200/build.py`` (called from
``__graft_entry__.build()``).  There is no fallback: if the library is missing, importing
the ops fails loudly.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
PRODUCT_SO = os.path.join(HERE, "libtfs.so")
# An A/B-timing variant (tools/build_variant.py) is loaded only when BOTH variables are set, so
# a stray TFS_LIB cannot silently replace the product; bench.py records which .so it loaded.
SO_PATH = (os.environ["TFS_LIB"] if os.environ.get("TFS_ALLOW_VARIANT_LIB") == "1"
           and os.environ.get("TFS_LIB") else PRODUCT_SO)
HEADER = os.path.join(os.path.dirname(HERE), "include", "tfs.h")

TFS_OK = 0
TFS_ERR_INVALID_ARGUMENT = 1
TFS_ERR_OUT_OF_RANGE = 2
TFS_ERR_BAD_POSITIONS = 3
TFS_ERR_WORKSPACE_TOO_SMALL = 4
TFS_ERR_CUDA = 5
TFS_ERR_UNSUPPORTED = 7
TFS_ERR_SAMPLER_EXHAUSTED = 8
TFS_ERR_CAPACITY = 9
TFS_ERR_COMM_TIMEOUT = 10
TFS_BF16_OPERANDS = 4
TFS_LABEL_IN_CANDIDATES = 8
TFS_F32, TFS_BF16 = 0, 1
TFS_SUBTRACT_LOG_Q, TFS_REMOVE_ACCIDENTAL_HITS = 1, 2

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
U32 = ctypes.c_uint32
U64 = ctypes.c_uint64
SZ = ctypes.c_size_t
F32 = ctypes.c_float


class TfsError(RuntimeError):
    def __init__(self, status: int, what: str, index: int = -1):
        self.status = status
        self.index = index
        msg = f"{what}: {status_string(status)} (status {status})"
        if index >= 0:
            msg += f" at input position {index}"
        if status == TFS_ERR_CUDA:
            msg += f" [{last_error_detail()}]"
        super().__init__(msg)


class SparseOpt(ctypes.Structure):
    _fields_ = [("kind", I32), ("lr", F32), ("mu", F32), ("slot", P), ("slot2", P),
                ("mirror", P)]


class StepConfigC(ctypes.Structure):
    _fields_ = [("vocab", I64), ("dim", I32), ("num_shards", I32), ("tokens", I64),
                ("num_sampled", I64), ("operand_dtype", I32), ("flags", U32), ("lr", F32),
                ("unique", I32), ("seed", U64), ("optimizer", I32), ("momentum", F32),
                ("adagrad_init", F32), ("cap_e", I64), ("cap_w", I64)]


class StepIO(ctypes.Structure):
    _fields_ = [("x", P), ("y", P), ("host", I32), ("loss_host", P), ("timing_events", P)]


class SsmArgs(ctypes.Structure):
    _fields_ = [
        ("B", I64), ("S", I64), ("dim", I32), ("operand_dtype", I32), ("flags", U32),
        ("grad_scale", F32),
        ("h", P), ("labels", P), ("w_true", P), ("b_true", P), ("log_ec_true", P),
        ("sampled", P), ("w_s", P), ("b_s", P), ("log_ec_s", P),
        ("loss", P), ("lse", P), ("loss_sum", P), ("dh", P), ("dw_true", P), ("db_true", P),
        ("dw_s", P), ("db_s", P), ("vocab", I64), ("timing_events", P), ("sm_reserve", I32),
        ("rows_ready_event", P),
    ]


_SIGNATURES = {
    "tfs_version": ([], I32),
    "tfs_ssm_grad_from_logits": ([], I32),
    "tfs_gather_peers2_bf16": ([P, I64, I32, P, P, I64, I64, I32, P, P, P, P], I32),
    "tfs_status_string": ([I32], ctypes.c_char_p),
    "tfs_last_error_detail": ([ctypes.c_char_p, SZ], I32),
    "tfs_device_check": ([I32], I32),
    "tfs_partition_workspace_bytes": ([I64, I32], SZ),
    "tfs_partition": ([P, I64, I64, I32, P, P, P, P, P, SZ, P, P], I32),
    "tfs_gather": ([P, I64, I32, I32, P, I64, P, I32, P, P], I32),
    "tfs_stitch_workspace_bytes": ([I64], SZ),
    "tfs_stitch": ([P, P, I64, I64, P, P, SZ, P, P], I32),
    "tfs_sampler_state_bytes": ([I64], SZ),
    "tfs_sampler_init": ([I64, I32, I32, P, ctypes.POINTER(I64), P], I32),
    "tfs_sampler_workspace_bytes": ([I64], SZ),
    "tfs_log_uniform_sample": ([P, I64, I32, I32, I64, U64, U64, P, U32, P, I64, P, P, P, P, P,
                                SZ, P, P], I32),
    "tfs_sample_commit": ([I64, I32, I32, P, P, P, P, I64, P, P, P, P, P, P, P], I32),
    "tfs_ssm_workspace_bytes": ([I64, I64, I32, I32, I64], SZ),
    "tfs_sampled_softmax_fwd_bwd": ([ctypes.POINTER(SsmArgs), P, SZ, P], I32),
    "tfs_ssm_partial_stats": ([ctypes.POINTER(SsmArgs), P, P, SZ, P], I32),
    "tfs_ssm_backward_from_lse": ([ctypes.POINTER(SsmArgs), P, P, SZ, P], I32),
    "tfs_lse_combine_peers": ([P, I32, I64, P, P], I32),
    "tfs_reduce_peers": ([P, I32, I64, I64, P, P], I32),
    "tfs_label_loss_sum": ([P, P, P, I64, I32, I32, F32, P, P], I32),
    "tfs_dense_sgd": ([P, P, I64, F32, P, P], I32),
    "tfs_sort_reduce_workspace_bytes": ([I64, I32], SZ),
    "tfs_sort_reduce": ([P, I64, I64, I32, P, I32, P, P, P, P, P, P, P, SZ, P, P], I32),
    "tfs_scatter_add_sgd_workspace_bytes": ([I64, I32], SZ),
    "tfs_scatter_add_sgd": ([P, I64, I32, P, P, I64, F32, P, P, P, SZ, P, P], I32),
    "tfs_scatter_plan_bytes": ([I64], SZ),
    "tfs_scatter_plan": ([P, I64, I64, P, SZ, P, P], I32),
    "tfs_scatter_apply_workspace_bytes": ([I64, I32], SZ),
    "tfs_scatter_add_sgd_planned": ([P, I64, I32, P, SZ, I64, P, F32, P, P, P, SZ, P], I32),
    "tfs_scatter_opt_planned": ([P, I64, I32, P, SZ, I64, P, P, P, ctypes.POINTER(SparseOpt), P,
                                 SZ, P], I32),
    "tfs_route_plan_bytes": ([I64, I32], SZ),
    "tfs_route_plan": ([P, I64, I64, I32, I64, P, SZ, P, I64, P, P, P], I32),
    "tfs_route_unpack": ([P, SZ, I64, I64, I32, I64, P, I64, I32, P, P], I32),
    "tfs_route_reduce_workspace_bytes": ([I64, I32], SZ),
    "tfs_route_reduce": ([P, SZ, I64, I64, I32, I64, P, I32, P, P, I64, P, I64, P, SZ, P], I32),
    "tfs_gather_slots": ([P, I64, I32, P, I64, I32, I64, P, I64, P, P], I32),
    "tfs_route_plan_push": ([P, I64, I64, I32, I64, P, SZ, P, I64, P, P, P], I32),
    "tfs_route_reduce_push": ([P, SZ, I64, I64, I32, I64, P, I32, P, P, I64, P, I64, P, SZ, P],
                              I32),
    "tfs_gather_peers": ([P, I64, I32, P, I64, I64, I32, P, I32, P, P], I32),
    "tfs_gather_peers2": ([P, I64, I32, P, P, I64, I64, I32, P, I32, P, P, P], I32),
    "tfs_gather2": ([P, I64, I32, P, P, I64, P, I32, P, P, P], I32),
    "tfs_scatter_plan_slots": ([P, I64, I32, I64, I64, I32, P, SZ, P, P], I32),
    "tfs_scatter_add_sgd_planned_slots": ([P, I64, I32, P, SZ, I32, I64, P, I64, F32, P, P, I64,
                                           P, SZ, P], I32),
    "tfs_scatter_opt_planned_slots": ([P, I64, I32, P, SZ, I32, I64, P, I64, P, P, I64,
                                       ctypes.POINTER(SparseOpt), P, SZ, P], I32),
    "tfs_comm_create": ([I32, I32, I32, I32, SZ, U32, ctypes.POINTER(P)], I32),
    "tfs_comm_export": ([P, P], I32),
    "tfs_comm_connect": ([P, P], I32),
    "tfs_comm_barrier": ([P, I32, P], I32),
    "tfs_comm_heap": ([P, I32], P),
    "tfs_comm_peer_bases": ([P, I32], P),
    "tfs_comm_error": ([P, I32], P),
    "tfs_comm_destroy": ([P], I32),
    "tfs_step_heap_bytes": ([ctypes.POINTER(StepConfigC)], SZ),
    "tfs_step_create": ([ctypes.POINTER(StepConfigC), P, ctypes.POINTER(P)], I32),
    "tfs_step_destroy": ([P], I32),
    "tfs_step_buffer": ([P, I32, I32, ctypes.POINTER(P), ctypes.POINTER(I64),
                         ctypes.POINTER(I32)], I32),
    "tfs_step_sync": ([P], I32),
    "tfs_step_set_counter": ([P, I64], I32),
    "tfs_step_run": ([P, ctypes.POINTER(StepIO), P], I32),
    "tfs_step_capture": ([P], I32),
    "tfs_step_uncapture": ([P], I32),
    "tfs_step_graph_kernels": ([P], I64),
    "tfs_debug_gemm_workspace_bytes": ([I32, I32, I32, I32], SZ),
    "tfs_debug_gemm_bf16": ([P, I64, I32, P, I64, I32, I32, I32, I32, I32, P, P, SZ, P], I32),
    "tfs_debug_launch_count": ([], I64),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libtfs.so (raises if it was not built -- no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(
                f"{SO_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
        L = ctypes.CDLL(SO_PATH)
        for name, (args, res) in _SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def status_string(status: int) -> str:
    return lib().tfs_status_string(status).decode()


def last_error_detail() -> str:
    buf = ctypes.create_string_buffer(512)
    lib().tfs_last_error_detail(buf, 512)
    return buf.value.decode(errors="replace")


def check(status: int, what: str):
    if status != TFS_OK:
        raise TfsError(status, what)
