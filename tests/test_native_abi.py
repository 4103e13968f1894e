"""The C-ABI boundary without a GPU: libsp_round.so loads (no torch types in
the interface, statically linked CUDA runtime) and exports every function
include/sp_round.h declares; the in-tree pybind module loads; the product
path refuses to run without the CUDA library (no CPU fallback)."""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_2106_10207_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    names = _declared("sp_round.h")
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native.EXPORTED_SYMBOLS)


def test_nm_dynamic_symbols_are_c_abi():
    from paper_2106_10207_b200 import _native

    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    for name in _declared("sp_round.h"):
        assert name in exported  # unmangled C symbols
    assert not any("torch" in s or "at::" in s for s in exported)


def test_version_and_error_channel():
    from paper_2106_10207_b200 import _native as nat

    L = nat.lib()
    assert b"sm_100a" in L.sp_version()
    h = ctypes.c_void_p()
    cfg = nat.SpRoundCfg(device=0, rank=0, world=1, peers_per_rank=1, n=0, wire=1)
    rc = L.sp_round_create(ctypes.byref(cfg), ctypes.byref(h))
    assert rc == nat.SP_ERR_ARG  # n = 0 rejected before touching the device
    assert b"n must be positive" in L.sp_last_error()
    with pytest.raises(ValueError):
        nat.check(rc)


def test_round_fails_loudly_without_library(tmp_path):
    code = ("import paper_2106_10207_b200._native as n; n.LIB_PATH = '/nonexistent/libsp_round.so';"
            "n._lib = None\ntry:\n n.lib()\nexcept RuntimeError as e:\n print('RAISED', e)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert "RAISED" in r.stdout and "no CPU fallback" in r.stdout


def test_swarmplan_module_loads_in_tree():
    from paper_2106_10207_b200 import _swarmplan

    assert _swarmplan.__file__.startswith(os.path.join(ROOT, "paper_2106_10207_b200"))
    assert _swarmplan.__version__ == "0.1.0"
