"""numpy/ctypes front of the CPU oracle (oracle/sp_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline and --impl reference). The product never imports it.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libsp_oracle.so")
WIRE = {"fp32": 0, "fp16": 1, "q8": 2}

_lib = None


class LambHP(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("bias_correction", ctypes.c_int)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from paper_2106_10207_b200 import _build
            _build.build_oracle()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.sp_oracle_f2h.restype = ctypes.c_uint16
        _lib.sp_oracle_f2h.argtypes = [ctypes.c_float]
        _lib.sp_oracle_h2f.restype = ctypes.c_float
        _lib.sp_oracle_h2f.argtypes = [ctypes.c_uint16]
        _lib.sp_oracle_splitmix64.restype = ctypes.c_uint64
        _lib.sp_oracle_splitmix64.argtypes = [ctypes.c_uint64]
        _lib.sp_oracle_fill_synthetic.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64,
                                                  ctypes.c_int, ctypes.c_float, ctypes.c_int64,
                                                  ctypes.c_float]
        _lib.sp_oracle_part_offsets.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                                ctypes.c_int64, ctypes.c_void_p]
        _lib.sp_oracle_pack_fp16.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        _lib.sp_oracle_pack_q8.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_int64, ctypes.c_int]
        _lib.sp_oracle_weighted_average_f64.argtypes = [ctypes.c_void_p, ctypes.c_void_p,
                                                        ctypes.c_int, ctypes.c_int64,
                                                        ctypes.c_void_p]
        _lib.sp_oracle_reduce.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_void_p]
        _lib.sp_oracle_lamb.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_int, ctypes.POINTER(LambHP), ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_void_p]
        _lib.sp_oracle_round.restype = ctypes.c_int
        _lib.sp_oracle_round.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_int, ctypes.POINTER(LambHP), ctypes.c_int,
                                         ctypes.c_int, ctypes.c_void_p]
        _lib.sp_oracle_max_threads.restype = ctypes.c_int
        _lib.sp_oracle_set_threads.argtypes = [ctypes.c_int]
        _lib.sp_oracle_wire_from_f64.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def fill_synthetic(n: int, seed: int, peer: int, scale: float, every: int = 997,
                   mult: float = 100.0) -> np.ndarray:
    out = np.empty(n, np.float32)
    lib().sp_oracle_fill_synthetic(_p(out), n, seed, peer, scale, every, mult)
    return out


def part_offsets(n: int, fractions, align: int) -> list[int]:
    f = np.ascontiguousarray(fractions, np.float64)
    out = np.empty(len(f) + 1, np.int64)
    lib().sp_oracle_part_offsets(n, len(f), _p(f), align, _p(out))
    return out.tolist()


def pack_fp16(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty(x.size, np.uint16)
    lib().sp_oracle_pack_fp16(_p(x), _p(out), x.size)
    return out


def pack_q8(x: np.ndarray, block: int):
    x = np.ascontiguousarray(x, np.float32)
    codes = np.empty(x.size, np.int8)
    scales = np.empty((x.size + block - 1) // block, np.float32)
    lib().sp_oracle_pack_q8(_p(x), _p(codes), _p(scales), x.size, block)
    return codes, scales


def pack(wire: str, x: np.ndarray, block: int = 4096):
    if wire == "fp32":
        return np.ascontiguousarray(x, np.float32), None
    if wire == "fp16":
        return pack_fp16(x), None
    return pack_q8(x, block)


def dequant(wire: str, buf: np.ndarray, scales: np.ndarray | None, block: int = 4096) -> np.ndarray:
    if wire == "fp32":
        return buf.astype(np.float32)
    if wire == "fp16":
        return buf.view(np.float16).astype(np.float32)
    s = np.repeat(scales, block)[: buf.size]
    return (buf.astype(np.float32) * s).astype(np.float32)


def weighted_average_f64(values: list[np.ndarray], weights) -> np.ndarray:
    vals = [np.ascontiguousarray(v, np.float64) for v in values]
    ptrs = (ctypes.c_void_p * len(vals))(*[v.ctypes.data for v in vals])
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    out = np.empty(vals[0].size, np.float64)
    lib().sp_oracle_weighted_average_f64(ptrs, _p(w), len(vals), vals[0].size, _p(out))
    return out


def reduce(wire: str, wires: list[np.ndarray], scales: list[np.ndarray | None], weights,
           lo: int, hi: int, n: int, block: int = 4096):
    """Returns (out_wire, out_scales) with elements [lo, hi) filled (rest zero)."""
    G = len(wires)
    wp = (ctypes.c_void_p * G)(*[w.ctypes.data for w in wires])
    sp = (ctypes.c_void_p * G)(*[0 if s is None else s.ctypes.data for s in scales])
    wt = np.ascontiguousarray(weights, np.float64)
    dtype = {"fp32": np.float32, "fp16": np.uint16, "q8": np.int8}[wire]
    out = np.zeros(n, dtype)
    osc = np.zeros((n + block - 1) // block, np.float32) if wire == "q8" else None
    lib().sp_oracle_reduce(WIRE[wire], wp, sp, _p(wt), G, lo, hi, block, _p(out), _p(osc))
    return out, osc


def lamb(wire: str, avg: np.ndarray, avg_scales, p, m, v, tensor_sizes, hp: dict, step: int,
         block: int = 4096, trust_in=None):
    """In-place LAMB on float32 p, m, v; returns the computed trust ratios."""
    ts = np.ascontiguousarray(tensor_sizes, np.int64)
    h = LambHP(hp["lr"], hp["beta1"], hp["beta2"], hp["eps"], hp["weight_decay"],
               int(hp.get("bias_correction", 1)))
    tout = np.empty(ts.size, np.float32)
    tin = None if trust_in is None else np.ascontiguousarray(trust_in, np.float32)
    lib().sp_oracle_lamb(WIRE[wire], _p(avg), _p(avg_scales), block, _p(p), _p(m), _p(v), p.size,
                         _p(ts), ts.size, ctypes.byref(h), step, _p(tin), _p(tout))
    return tout


def round_cpu(wire: str, grads: list[np.ndarray], weights, p, m, v, tensor_sizes, hp: dict,
              step: int, block: int = 4096, threads: int = 0):
    G = len(grads)
    gp = (ctypes.c_void_p * G)(*[0 if g is None else g.ctypes.data for g in grads])
    wt = np.ascontiguousarray(weights, np.float64)
    ts = np.ascontiguousarray(tensor_sizes, np.int64)
    h = LambHP(hp["lr"], hp["beta1"], hp["beta2"], hp["eps"], hp["weight_decay"],
               int(hp.get("bias_correction", 1)))
    tout = np.empty(ts.size, np.float32)
    lib().sp_oracle_round(WIRE[wire], block, G, p.size, gp, _p(wt), _p(p), _p(m), _p(v), _p(ts),
                          ts.size, ctypes.byref(h), step, threads, _p(tout))
    return tout


def max_threads() -> int:
    return int(lib().sp_oracle_max_threads())


def set_threads(threads: int) -> None:
    lib().sp_oracle_set_threads(int(threads))


def wire_from_f64(wire: str, x: np.ndarray, block: int = 4096):
    """fp64 -> fp32 -> wire format; returns (values, scales) like pack()."""
    x = np.ascontiguousarray(x, np.float64)
    dtype = {"fp32": np.float32, "fp16": np.uint16, "q8": np.int8}[wire]
    out = np.empty(x.size, dtype)
    sc = np.empty((x.size + block - 1) // block, np.float32) if wire == "q8" else None
    lib().sp_oracle_wire_from_f64(WIRE[wire], _p(x), _p(out), _p(sc), x.size, block)
    return out, sc
