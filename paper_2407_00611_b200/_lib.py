"""ctypes loader of the in-tree libwf.so (the C ABI of include/wf.h).

Fails loudly when the library is missing: there is no CPU or Python fallback.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WF_LIB_PATH") or os.path.join(_HERE, "libwf.so")

c_int, c_i64, c_p, c_f = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_float
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i64p = ctypes.POINTER(ctypes.c_int64)


class WfUid(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_uint8 * 128)]


class WfEvent(ctypes.Structure):
    _fields_ = [("pas", ctypes.c_int32), ("kind", ctypes.c_int32), ("step", ctypes.c_int32),
                ("src", ctypes.c_int32), ("dst", ctypes.c_int32), ("block", ctypes.c_int32),
                ("nbytes", ctypes.c_int64)]


KINDS = ["AG_Q", "AG_KV", "INIT_KV", "SLICE_KV", "RING_KV", "RS_O", "RS_LSE", "AG_QDO", "AG_STATS",
         "RING_QPKG", "RING_DQ", "RET_DQ", "REV_DKV", "RS_DKV", "RS_DQ"]

_SIGS = {
    "wf_get_uid": (c_int, [ctypes.POINTER(WfUid)]),
    "wf_init": (c_int, [c_int, c_int, c_int, c_int, ctypes.POINTER(WfUid), ctypes.POINTER(c_p)]),
    "wf_init_emulated": (c_int, [c_int, c_int, ctypes.POINTER(c_p)]),
    "wf_init_bootstrap": (c_int, [c_int, c_int, c_int, c_int, c_p, c_p, ctypes.POINTER(c_p)]),
    "wf_set_timeout": (c_int, [c_p, ctypes.c_double]),
    "wf_attn_fwd": (c_int, [c_p, c_p, c_p, c_p, c_i64, c_int, c_int, c_int, c_p, c_p, c_p]),
    "wf_qkv_proj": (c_int, [c_p, c_p, c_p, c_i64, c_int, c_int, c_int, c_int, c_p, c_p, c_p, c_p]),
    "wf_gemm_bf16": (c_int, [c_p, c_p, c_int, c_int, c_int, c_p, c_p]),
    "wf_gemm_bf16_t": (c_int, [c_p, c_int, c_p, c_int, c_int, c_int, c_int, c_p, c_p]),
    "wf_layernorm_fwd": (c_int, [c_p, c_p, c_p, c_i64, c_int, ctypes.c_float, c_p, c_p, c_p, c_p]),
    "wf_layernorm_bwd": (c_int, [c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_int, c_p, c_p, c_p, c_p]),
    "wf_gelu_fwd": (c_int, [c_p, c_i64, c_p, c_p]),
    "wf_gelu_bwd": (c_int, [c_p, c_p, c_i64, c_p, c_p]),
    "wf_add_bf16": (c_int, [c_p, c_p, c_i64, c_p, c_p]),
    "wf_pack3_bf16": (c_int, [c_p, c_p, c_p, c_i64, c_int, c_p, c_p]),
    "wf_attn_bwd": (c_int, [c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_int, c_int, c_int, c_p, c_p, c_p, c_p]),
    "wf_get_trace": (c_int, [c_p, ctypes.POINTER(WfEvent), ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "wf_plan_trace": (c_int, [c_int, c_int, c_i64, c_int, c_int, c_int, ctypes.POINTER(WfEvent), ctypes.c_size_t,
                              ctypes.POINTER(ctypes.c_size_t)]),
    "wf_plan": (c_int, [c_int, c_int, c_int, c_i32p]),
    "wf_set_schedule": (c_int, [c_p, c_int]),
    "wf_plan_trace_sched": (c_int, [c_int, c_int, c_i64, c_int, c_int, c_int, c_int, ctypes.POINTER(WfEvent),
                                    ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "wf_workspace_bytes": (c_int, [c_int, c_int, c_i64, c_int, c_int, c_int, ctypes.POINTER(ctypes.c_size_t)]),
    "wf_shard_ranges": (c_int, [c_int, c_int, c_i64, c_int, c_i64p]),
    "wf_kernel_launches": (c_i64, [c_p]),
    "wf_set_profiling": (c_int, [c_p, c_int]),
    "wf_set_debug": (c_int, [c_p, c_int]),
    "wf_phase_times": (c_int, [c_p, ctypes.POINTER(ctypes.c_double), c_int]),
    "wf_kernel_times": (c_int, [c_p, ctypes.POINTER(ctypes.c_double)]),
    "wf_debug_timeline": (c_int, [c_int]),
    "wf_debug_timeline_read": (c_int, [ctypes.POINTER(ctypes.c_uint64), ctypes.c_size_t]),
    "wf_last_error": (ctypes.c_char_p, [c_p]),
    "wf_finalize": (c_int, [c_p]),
    "wf_block_fwd": (c_int, [c_p, c_p, c_p, c_int, c_int, c_int, c_int, c_int, c_int, c_i32p, c_int, c_i32p, c_int,
                             c_p, c_p, c_p, c_p, c_p, c_p]),
    "wf_block_bwd": (c_int, [c_p, c_p, c_p, c_p, c_p, c_p, c_int, c_int, c_int, c_int, c_int, c_int, c_i32p, c_int,
                             c_i32p, c_int, c_p, c_p, c_p, c_int, c_p]),
}

EXPORTED = sorted(_SIGS)

# int (*wf_allgather_fn)(const void* in, void* out, size_t bytes, void* user)
ALLGATHER_FN = ctypes.CFUNCTYPE(c_int, c_p, c_p, ctypes.c_size_t, c_p)


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(f"libwf.so not built ({path}); run `python -m paper_2407_00611_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = load()
    return _lib
