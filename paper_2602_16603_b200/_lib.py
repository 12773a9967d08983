"""ctypes binding of the C ABI declared in include/flowprefill.h.

The shared library is built in-tree (``__graft_entry__.build()`` / ``python -m
paper_2602_16603_b200.build``) into ``paper_2602_16603_b200/_native/libflowprefill.so``.
There is no fallback: if the library is missing or fails to load, every GPU entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_native", "libflowprefill.so")
# A/B experiments only: another build of the library (symbols it lacks stay unbound)
_AB_PATH = os.environ.get("FP_AB_LIB")

FP_OK = 0
FP_GRAN = {"operator": 0, "layer": 1, "chunk": 2, "none": 3}
FP_TASK_IDLE, FP_TASK_RUNNING, FP_TASK_STOPPED, FP_TASK_DONE = 0, 1, 2, 3

W_EMBED, W_Q, W_K, W_V, W_O, W_GATE, W_UP, W_DOWN = range(8)
W_ATTN_NORM, W_FFN_NORM, W_FINAL_NORM, W_LM_HEAD = 8, 9, 10, 11
W_Q_BIAS, W_K_BIAS, W_V_BIAS, W_Q_NORM, W_K_NORM = 12, 13, 14, 15, 16
W_ROUTER, W_EXPERT_GATE, W_EXPERT_UP, W_EXPERT_DOWN = 17, 18, 19, 20


class NativeError(RuntimeError):
    """A C-ABI call returned a negative status."""


class ModelCfg(C.Structure):
    _fields_ = [
        ("num_layers", C.c_int32),
        ("hidden", C.c_int32),
        ("n_heads", C.c_int32),
        ("n_kv_heads", C.c_int32),
        ("head_dim", C.c_int32),
        ("ffn", C.c_int32),
        ("vocab", C.c_int32),
        ("max_pos", C.c_int32),
        ("rope_theta", C.c_float),
        ("rms_eps", C.c_float),
        ("qkv_bias", C.c_int32),
        ("qk_norm", C.c_int32),
        ("n_experts", C.c_int32),
        ("top_k", C.c_int32),
        ("moe_ffn", C.c_int32),
        ("norm_topk", C.c_int32),
    ]


class Status(C.Structure):
    _fields_ = [
        ("ack_seq", C.c_int32),
        ("ack_task", C.c_int32),
        ("ack_entry", C.c_int32),
        ("progress_task", C.c_int32),
        ("progress_entry", C.c_int32),
        ("signal", C.c_int32),
        ("ack_ns", C.c_uint64),
    ]


class TaskStatus(C.Structure):
    _fields_ = [
        ("state", C.c_int32),
        ("cursor", C.c_int32),
        ("generation", C.c_int32),
        ("enqueued", C.c_int32),
    ]


class TaskInfo(C.Structure):
    _fields_ = [
        ("n_entries", C.c_int32),
        ("n_chunks", C.c_int32),
        ("n_seqs", C.c_int32),
        ("total_tokens", C.c_int32),
        ("max_chunk_tokens", C.c_int32),
        ("n_pages", C.c_int32),
        ("upload_bytes", C.c_int64),
    ]


class ProfRec(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("layer", C.c_int32),
        ("M", C.c_int32),
        ("pad", C.c_int32),
        ("flops", C.c_double),
        ("bytes", C.c_double),
        ("ms", C.c_double),
    ]


KERNEL_KINDS = ("rmsnorm", "qkv_gemm", "attn", "o_gemm", "gate_up_gemm", "down_gemm",
                "lm_head_gemm", "final_rmsnorm", "tp_allreduce", "router_gemm", "moe_dispatch",
                "expert_gate_up_gemm", "expert_down_gemm", "moe_combine")


class TpHandle(C.Structure):
    """fp_tp_handle: one rank's exported exchange block (include/flowprefill.h)."""

    _fields_ = [
        ("ipc", C.c_char * 64),
        ("part_rows", C.c_int64),
        ("rank", C.c_int32),
        ("device", C.c_int32),
    ]

# name -> (restype, argtypes)
_P = C.c_void_p
_I = C.c_int32
_SIGS = {
    "fp_last_error": (C.c_char_p, []),
    "fp_version": (C.c_int, []),
    "fp_ctx_create": (C.c_int, [_I, C.POINTER(ModelCfg), _I, _I, _P, C.c_int64, _I, C.POINTER(_P)]),
    "fp_ctx_destroy": (C.c_int, [_P]),
    "fp_ctx_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "fp_ctx_free_pages": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "fp_ctx_set_window": (C.c_int, [_P, _I]),
    "fp_ctx_set_gemm_policy": (C.c_int, [_P, _I, _I]),
    "fp_ctx_set_skinny_max": (C.c_int, [_P, _I]),
    "fp_ctx_set_batch_invariant": (C.c_int, [_P, _I]),
    "fp_task_read_routing": (C.c_int, [_P, _P, _P, _P, _I]),
    "fp_op_gate_up_swiglu": (C.c_int, [_P, _P, _P, _P, _P, _I, _I, _I]),
    "fp_op_qkv_rope_kv": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I]),
    "fp_op_tp_allreduce": (C.c_int, [_P, _I, _P, _P, _I]),
    "fp_op_attn_prefill": (C.c_int, [_P, _P, _P, _P, _P, _I, _I]),
    "fp_debug_gemm_stamps": (C.c_int, [_P, _P, _I]),
    "fp_sync": (C.c_int, [_P]),
    "fp_weights_init_random": (C.c_int, [_P, C.c_uint64, C.c_float]),
    "fp_weights_load": (C.c_int, [_P, _I, _I, _P, C.c_int64]),
    "fp_task_create": (C.c_int, [_P, _P, _P, _I, _I, _I, _I, C.POINTER(_P)]),
    "fp_task_num_entries": (C.c_int, [_P]),
    "fp_task_info": (C.c_int, [_P, C.POINTER(TaskInfo)]),
    "fp_task_entry_info": (C.c_int, [_P, _I, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    "fp_task_destroy": (C.c_int, [_P, _P]),
    "fp_task_begin_segment": (C.c_int, [_P, _P, _I]),
    "fp_task_enqueue": (C.c_int, [_P, _P, _I, _I]),
    "fp_task_start": (C.c_int, [_P, _P, _I]),
    "fp_task_poll": (C.c_int, [_P, _P, C.POINTER(TaskStatus)]),
    "fp_signal": (C.c_int, [_P]),
    "fp_clear": (C.c_int, [_P]),
    "fp_poll": (C.c_int, [_P, C.POINTER(Status)]),
    "fp_task_logits": (C.c_int, [_P, _P, _P]),
    "fp_task_entry_stamps": (C.c_int, [_P, _P, _P]),
    "fp_task_read_kv": (C.c_int, [_P, _P, _I, _I, _P, _P]),
    "fp_prof_enable": (C.c_int, [_P, _I]),
    "fp_prof_collect": (C.c_int, [_P, C.POINTER(ProfRec), _I, C.POINTER(_I)]),
    "fp_ctx_launch_count": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "fp_tp_export": (C.c_int, [_P, C.c_int64, C.POINTER(TpHandle)]),
    "fp_tp_import": (C.c_int, [_P, C.POINTER(TpHandle)]),
    "fp_tp_connect_local": (C.c_int, [C.POINTER(_P), _I, C.c_int64]),
    "fp_tp_enqueue_lockstep": (C.c_int, [C.POINTER(_P), C.POINTER(_P), _I, _I, _I]),
    "fp_ctx_tp_counters": (C.c_int, [_P, C.POINTER(_I)]),
    "fp_op_gemm": (C.c_int, [_P, _I, _P, _P, _P, _I, _I, _I]),
    "fp_op_rmsnorm": (C.c_int, [_P, _P, _P, _P, _I, _I, C.c_float]),
}

_lib: Optional[C.CDLL] = None


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load (once) and type the native library. Raises if it is absent: no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if _AB_PATH:
        path = _AB_PATH
    if not os.path.exists(path):
        raise NativeError(
            f"native library missing: {path}. Build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a)."
        )
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        if _AB_PATH and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc != FP_OK:
        msg = load().fp_last_error().decode(errors="replace")
        raise NativeError(f"{what or 'native call'} failed ({rc}): {msg}")
