"""ctypes binding of libsp_round.so (include/sp_round.h).

This is the Python side of the C-ABI boundary: plain pointers and sizes go
in, SP_* status codes come back and are mapped onto the exception classes
the reference raises (std::invalid_argument -> ValueError,
std::runtime_error -> RuntimeError; /root/reference/proj/src/groups.cpp:44-46,
/root/reference/proj/src/strategy.cpp:325). There is no fallback: a missing
or unloadable library raises immediately.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libsp_round.so")

SP_OK, SP_ERR_ARG, SP_ERR_CUDA, SP_ERR_STATE, SP_ERR_PEER, SP_ERR_SHAPE = range(6)
SP_WIRE_FP32, SP_WIRE_FP16, SP_WIRE_Q8 = range(3)
SP_BUF_WIRE, SP_BUF_AVG, SP_BUF_TRUST = range(3)
WIRE_FORMATS = {"fp32": SP_WIRE_FP32, "fp16": SP_WIRE_FP16, "q8": SP_WIRE_Q8}


class SpRoundCfg(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int),
        ("rank", ctypes.c_int),
        ("world", ctypes.c_int),
        ("peers_per_rank", ctypes.c_int),
        ("n", ctypes.c_int64),
        ("wire", ctypes.c_int),
        ("q8_block", ctypes.c_int),
        ("num_tensors", ctypes.c_int),
        ("tensor_sizes", ctypes.POINTER(ctypes.c_int64)),
        ("lr", ctypes.c_float),
        ("beta1", ctypes.c_float),
        ("beta2", ctypes.c_float),
        ("eps", ctypes.c_float),
        ("weight_decay", ctypes.c_float),
        ("bias_correction", ctypes.c_int),
        ("barrier_timeout_s", ctypes.c_double),
        ("shard_lamb", ctypes.c_int),
    ]


class SpPhaseTimes(ctypes.Structure):
    _fields_ = [(k, ctypes.c_float) for k in (
        "pack_ms", "barrier_a_ms", "reduce_ms", "barrier_b_ms", "lamb_ms", "barrier_c_ms",
        "total_ms")]


class SpPlanDesc(ctypes.Structure):
    _fields_ = [
        ("pack_ranges", ctypes.c_int),
        ("pack_owner", ctypes.c_int * 8),
        ("pack_first_unit", ctypes.c_int64 * 8),
        ("pack_units", ctypes.c_int64 * 8),
        ("pack_cta_begin", ctypes.c_int * 9),
        ("pack_ctas", ctypes.c_int),
        ("unit_elems", ctypes.c_int),
        ("own_lo", ctypes.c_int64),
        ("own_hi", ctypes.c_int64),
        ("push_order", ctypes.c_int * 8),
        ("avg_push_ranks", ctypes.c_int),
    ]


class PeerTimeout(RuntimeError):
    """A cross-rank barrier timed out (a peer process died or stalled)."""


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback for the averaging round)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    sig = {
        "sp_round_create": (c_int, [ctypes.POINTER(SpRoundCfg), ctypes.POINTER(vp)]),
        "sp_round_destroy": (c_int, [vp]),
        "sp_round_handle_bytes": (ctypes.c_size_t, []),
        "sp_round_export": (c_int, [vp, vp]),
        "sp_round_connect": (c_int, [vp, vp]),
        "sp_round_align": (c_int, [vp]),
        "sp_round_set_assignment": (c_int, [vp, ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double)]),
        "sp_round_run": (c_int, [vp, ctypes.POINTER(vp), vp, vp, vp, c_int, vp]),
        "sp_round_run_host": (c_int, [vp, ctypes.POINTER(vp), vp, vp, vp, c_int, vp]),
        "sp_round_run_host_params": (c_int, [vp, ctypes.POINTER(vp), vp, vp, vp, c_int, vp, vp]),
        "sp_round_run_phased": (c_int, [vp, ctypes.POINTER(vp), vp, vp, vp, c_int, vp,
                                        ctypes.POINTER(SpPhaseTimes)]),
        "sp_round_wire_ptr": (vp, [vp, c_int]),
        "sp_round_avg_ptr": (vp, [vp]),
        "sp_round_param_ptr": (vp, [vp]),
        "sp_round_lamb_chunks": (c_int, [vp, ctypes.POINTER(c_int)]),
        "sp_round_describe": (c_int, [ctypes.POINTER(SpRoundCfg), ctypes.POINTER(i64), c_int,
                                      ctypes.POINTER(SpPlanDesc)]),
        "sp_round_padded_n": (i64, [vp]),
        "sp_round_trust_ptr": (vp, [vp]),
        "sp_round_copy_trust": (c_int, [vp, vp, vp]),
        "sp_round_read": (c_int, [vp, c_int, c_int, ctypes.c_size_t, vp, ctypes.c_size_t]),
        "sp_round_accumulate": (c_int, [vp, c_int, c_int, vp, ctypes.c_double, vp]),
        "sp_round_accumulator_ptr": (vp, [vp, c_int, c_int]),
        "sp_round_add_samples": (c_int, [vp, c_int, c_int, ctypes.c_double]),
        "sp_round_samples": (ctypes.c_double, [vp, c_int, c_int]),
        "sp_round_run_accumulated": (c_int, [vp, c_int, vp, vp, vp, c_int, vp]),
        "sp_vec_scale": (c_int, [vp, vp, ctypes.c_double, i64, vp]),
        "sp_vec_sum": (c_int, [vp, ctypes.POINTER(vp), c_int, i64, vp]),
        "sp_vec_div": (c_int, [vp, vp, ctypes.c_double, i64, vp]),
        "sp_fill_synthetic": (c_int, [vp, i64, ctypes.c_uint64, c_int, ctypes.c_float, i64,
                                      ctypes.c_float, vp]),
        "sp_version": (ctypes.c_char_p, []),
        "sp_last_error": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTED_SYMBOLS = [
    "sp_round_create", "sp_round_destroy", "sp_round_handle_bytes", "sp_round_export",
    "sp_round_connect", "sp_round_align", "sp_round_set_assignment", "sp_round_run",
    "sp_round_run_host", "sp_round_run_host_params", "sp_round_run_phased", "sp_round_wire_ptr",
    "sp_round_avg_ptr", "sp_round_param_ptr", "sp_round_lamb_chunks", "sp_round_describe", "sp_round_padded_n",
    "sp_round_trust_ptr", "sp_round_copy_trust", "sp_round_read", "sp_round_accumulate", "sp_round_accumulator_ptr",
    "sp_round_add_samples", "sp_round_samples", "sp_round_run_accumulated",
    "sp_vec_scale", "sp_vec_sum", "sp_vec_div", "sp_fill_synthetic", "sp_version", "sp_last_error",
]


def check(rc: int) -> None:
    if rc == SP_OK:
        return
    msg = lib().sp_last_error().decode(errors="replace")
    if rc in (SP_ERR_ARG, SP_ERR_SHAPE):
        raise ValueError(msg)
    if rc == SP_ERR_PEER:
        raise PeerTimeout(msg)
    raise RuntimeError(msg)
