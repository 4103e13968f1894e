"""ctypes front of oracle/_ref/libswarmplan_ref.so: the reference's own
groups.cpp / model.cpp compiled by oracle/build_ref.py.

TEST INFRASTRUCTURE ONLY: imported by tests/ and by bench.py's reference arm
(--impl reference). The product never imports it.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libswarmplan_ref.so")
_lib = None


def available() -> bool:
    if os.path.exists(LIB_PATH):
        return True
    from oracle import build_ref

    return build_ref.build() is not None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{LIB_PATH} missing and /root/reference absent (oracle/build_ref.py)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_build_plan.argtypes = [c_int, c_int, vp, c_int]
        L.ref_run_plan.argtypes = [c_int, c_int, vp, i64, vp, c_int, vp, c_int, vp, vp, vp, vp]
        L.ref_validate.argtypes = [ctypes.c_char_p, vp, c_int]
        L.ref_spec_roundtrip.argtypes = [ctypes.c_char_p, vp, c_int]
        L.ref_assignment_json.argtypes = [ctypes.c_char_p, c_int, vp, vp, vp, vp, vp, ctypes.c_double,
                                          c_int, vp, c_int]
        L.ref_weighted_mean.argtypes = [c_int, vp, vp, i64, i64, vp]
        L.ref_weighted_mean_wire.argtypes = [c_int, c_int, vp, vp, c_int, vp, i64, i64, c_int, vp]
        _lib = L
    return _lib


def _err() -> str:
    return lib().ref_last_error().decode()


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def build_plan(n: int, m: int) -> list:
    cap = 64 + 4 * n * (n + 8)
    buf = np.empty(cap, np.int32)
    k = lib().ref_build_plan(n, m, _p(buf), cap)
    if k == -1:
        raise ValueError(_err())
    if k < 0:
        raise RuntimeError("ref_build_plan: buffer too small")
    it = iter(buf[:k].tolist())
    rounds = []
    for _ in range(next(it)):
        groups = []
        for _ in range(next(it)):
            size = next(it)
            groups.append([next(it) for _ in range(size)])
        rounds.append(groups)
    return rounds


def run_plan(n: int, m: int, values: np.ndarray, weights=(), failures=()) -> dict:
    v = np.ascontiguousarray(values, np.float64)
    if v.ndim != 2:
        raise ValueError("values must be 2-D")
    dim = v.shape[1]
    w = np.ascontiguousarray(weights, np.float64) if len(weights) else None
    f = np.ascontiguousarray(np.asarray(failures, np.int32).reshape(-1), np.int32)
    out = np.empty((n, dim), np.float64)
    comp = np.empty(n, np.int32)
    cov = np.empty(n, np.int32)
    gf = ctypes.c_int(0)
    rc = lib().ref_run_plan(n, m, _p(v), dim, _p(w), 0 if w is None else w.size, _p(f), len(failures),
                            _p(out), _p(comp), _p(cov), ctypes.byref(gf))
    if rc == -1:
        raise ValueError(_err())
    if rc:
        raise RuntimeError(_err())
    return {"values": out, "complete": [bool(x) for x in comp], "coverage": cov.tolist(),
            "groups_failed": gf.value}


def validate(spec_json: str) -> list[tuple[int, str, str]]:
    cap = 1 << 20
    buf = ctypes.create_string_buffer(cap)
    k = lib().ref_validate(spec_json.encode(), buf, cap)
    if k == -1:
        raise ValueError(_err())
    lines = buf.value.decode().splitlines()
    return [(int(a), b, c) for a, b, c in (ln.split("\t", 2) for ln in lines)]


def spec_roundtrip(spec_json: str) -> str:
    cap = 1 << 22
    buf = ctypes.create_string_buffer(cap)
    k = lib().ref_spec_roundtrip(spec_json.encode(), buf, cap)
    if k == -1:
        raise ValueError(_err())
    return buf.value.decode()


def assignment_json(spec_json: str, a, g, c_raw, compute, fractions, xi: float, lp_iterations: int) -> str:
    n = len(fractions)
    A = np.ascontiguousarray(a, np.float64).reshape(n, n)
    Gm = np.ascontiguousarray(g, np.float64).reshape(n, n)
    c = np.ascontiguousarray(c_raw, np.float64)
    cm = np.ascontiguousarray([1 if x else 0 for x in compute], np.int32)
    fr = np.ascontiguousarray(fractions, np.float64)
    cap = 1 << 22
    buf = ctypes.create_string_buffer(cap)
    k = lib().ref_assignment_json(spec_json.encode(), n, _p(A), _p(Gm), _p(c), _p(cm), _p(fr), float(xi),
                                  int(lp_iterations), buf, cap)
    if k < 0:
        raise RuntimeError(_err())
    return buf.value.decode()


def weighted_mean(rows: list, weights, block: int = 1 << 16) -> np.ndarray:
    """The reference's run_plan at m = n (one group of all G peers) over fp32
    rows (None = a weight-0 peer): the fp64 weighted mean, peer order."""
    G = len(rows)
    N = next(r.size for r in rows if r is not None)
    keep = [None if r is None else np.ascontiguousarray(r, np.float32) for r in rows]
    ptrs = (ctypes.c_void_p * G)(*[0 if r is None else r.ctypes.data for r in keep])
    w = np.ascontiguousarray(weights, np.float64)
    out = np.empty(N, np.float64)
    rc = lib().ref_weighted_mean(G, ptrs, _p(w), N, block, _p(out))
    if rc:
        raise RuntimeError(_err())
    return out


WIRE = {"fp32": 0, "fp16": 1, "q8": 2}


def weighted_mean_wire(wire: str, packed: list, weights, qblock: int = 4096, threads: int = 1,
                       block: int = 1 << 16, out: np.ndarray | None = None) -> np.ndarray:
    """The reference's run_plan weighted mean (m = n) over the peers' wire
    buffers: `packed` holds (values, scales) per peer (None for a weight-0
    peer), as oracle.oracle.pack returns them. Column blocks are spread over
    `threads` threads, each running the reference's own run_plan."""
    G = len(packed)
    N = next(q[0].size for q in packed if q is not None)
    rows = (ctypes.c_void_p * G)(*[0 if q is None else q[0].ctypes.data for q in packed])
    scl = (ctypes.c_void_p * G)(*[0 if q is None or q[1] is None else q[1].ctypes.data for q in packed])
    w = np.ascontiguousarray(weights, np.float64)
    if out is None:
        out = np.empty(N, np.float64)
    rc = lib().ref_weighted_mean_wire(WIRE[wire], G, rows, scl, qblock, _p(w), N, block, threads, _p(out))
    if rc:
        raise RuntimeError(_err())
    return out
