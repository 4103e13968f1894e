"""In-tree native build: nvcc/g++ straight to .so files next to the sources.

Outputs (git-ignored, shipped to the GPU box by gpurun's snapshot):
  paper_2106_10207_b200/lib/libsp_round.so   CUDA executor + C-ABI (sm_100a)
  paper_2106_10207_b200/lib/libswarmplan.so  host C++ (LP, strategy, groups, round)
  paper_2106_10207_b200/_swarmplan*.so       pybind11 module (reference API)
  oracle/_build/libsp_oracle.so              CPU oracle (test infrastructure)
  tests/cpp/_build/unit_tests                C++ unit tests of the host API

No JIT cache, no torch extension machinery: the .so files are plain shared
libraries so the product path can be loaded without torch.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
import sysconfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2106_10207_b200")
LIB = os.path.join(PKG, "lib")
INC = os.path.join(ROOT, "include")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]

CUDA_SOURCES = [os.path.join(PKG, "csrc", "cuda", "sp_round.cu")]
CUDA_DEPS = CUDA_SOURCES + glob.glob(os.path.join(PKG, "csrc", "cuda", "*.cuh")) + glob.glob(
    os.path.join(PKG, "csrc", "cuda", "*.h")) + [
    os.path.join(INC, "sp_round.h")
]
HOST_SOURCES = sorted(glob.glob(os.path.join(PKG, "csrc", "host", "*.cpp")))
HOST_DEPS = HOST_SOURCES + glob.glob(os.path.join(INC, "swarmplan", "*.hpp")) + [
    os.path.join(INC, "sp_round.h")
]
BIND_SOURCES = [os.path.join(PKG, "csrc", "bindings", "module.cpp")]
ORACLE_SOURCES = [os.path.join(ROOT, "oracle", "sp_oracle.c")]
ORACLE_DEPS = ORACLE_SOURCES + [os.path.join(ROOT, "oracle", "sp_oracle.h")]
TEST_SOURCES = sorted(glob.glob(os.path.join(ROOT, "tests", "cpp", "*.cpp")))


def _json_include() -> str:
    """nlohmann/json (third-party, header-only; ships inside the image)."""
    for cand in glob.glob(
        os.path.join(sys.prefix, "lib", "python3*", "site-packages", "include",
                     "cudnn_frontend", "thirdparty")
    ) + ["/usr/include", "/usr/local/include"]:
        if os.path.exists(os.path.join(cand, "nlohmann", "json.hpp")):
            return cand
    raise RuntimeError("nlohmann/json.hpp not found")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd: list[str]) -> None:
    print("[build]", " ".join(os.path.relpath(c, ROOT) if c.startswith(ROOT) else c
                              for c in cmd), flush=True)
    subprocess.run(cmd, check=True)


def build_cuda(force: bool = False) -> str:
    out = os.path.join(LIB, "libsp_round.so")
    if force or _stale(out, CUDA_DEPS):
        os.makedirs(LIB, exist_ok=True)
        _run([NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-Wall", "-shared", f"-I{INC}", "-o", out, *CUDA_SOURCES])
    return out


def build_oracle(force: bool = False) -> str:
    out = os.path.join(ROOT, "oracle", "_build", "libsp_oracle.so")
    if force or _stale(out, ORACLE_DEPS):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        _run(["gcc", "-O3", "-mavx2", "-mfma", "-ffp-contract=off", "-fno-fast-math",
              "-fopenmp", "-fPIC", "-shared", "-Wall", "-Wextra", "-o", out,
              *ORACLE_SOURCES, "-lm"])
    return out


def _host_flags() -> list[str]:
    # x86-64-v3 (AVX2/FMA): every B200 host CPU has it; 1.3x on the LP
    return ["-O3", "-march=x86-64-v3", "-std=c++20", "-fPIC", "-Wall", "-Wextra", f"-I{INC}",
            f"-I{_json_include()}", f"-I{os.path.join(CUDA_HOME, 'include')}"]


def build_host(force: bool = False) -> str:
    out = os.path.join(LIB, "libswarmplan.so")
    if not HOST_SOURCES:
        return out
    if force or _stale(out, HOST_DEPS + [os.path.join(LIB, "libsp_round.so")]):
        _run(["g++", *_host_flags(), "-shared", "-o", out, *HOST_SOURCES,
              f"-L{LIB}", "-lsp_round", f"-L{os.path.join(CUDA_HOME, 'lib64')}", "-lcudart",
              f"-Wl,-rpath,$ORIGIN:{os.path.join(CUDA_HOME, 'lib64')}"])
    return out


def build_bindings(force: bool = False) -> str | None:
    if not os.path.exists(BIND_SOURCES[0]):
        return None
    import pybind11

    suffix = sysconfig.get_config_var("EXT_SUFFIX")
    out = os.path.join(PKG, "_swarmplan" + suffix)
    if force or _stale(out, BIND_SOURCES + HOST_DEPS + [os.path.join(LIB, "libswarmplan.so")]):
        _run(["g++", *_host_flags(), "-shared", f"-I{pybind11.get_include()}",
              f"-I{sysconfig.get_paths()['include']}", "-o", out, *BIND_SOURCES,
              f"-L{LIB}", "-lswarmplan", "-lsp_round", "-Wl,-rpath,$ORIGIN/lib"])
    return out


def build_tests(force: bool = False) -> str | None:
    if not TEST_SOURCES:
        return None
    out = os.path.join(ROOT, "tests", "cpp", "_build", "unit_tests")
    if force or _stale(out, TEST_SOURCES + HOST_DEPS + [os.path.join(LIB, "libswarmplan.so")]):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        _run(["g++", *_host_flags(), "-o", out, *TEST_SOURCES, f"-L{LIB}", "-lswarmplan",
              "-lsp_round", f"-Wl,-rpath,{LIB}"])
    return out


def build_gpu_tests(force: bool = False) -> str | None:
    """C++ GPU check of the orchestrator (run by tests/test_cpp_gpu.py on a B200)."""
    src = os.path.join(ROOT, "tests", "cpp_gpu", "round_check.cpp")
    if not os.path.exists(src):
        return None
    out = os.path.join(ROOT, "tests", "cpp_gpu", "_build", "round_check")
    deps = [src] + HOST_DEPS + ORACLE_DEPS + [os.path.join(LIB, "libswarmplan.so")]
    if force or _stale(out, deps):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        oracle_dir = os.path.join(ROOT, "oracle", "_build")
        _run(["g++", *_host_flags(), "-o", out, src, f"-L{LIB}", "-lswarmplan", "-lsp_round",
              f"-L{oracle_dir}", "-lsp_oracle", f"-L{os.path.join(CUDA_HOME, 'lib64')}", "-lcudart",
              f"-Wl,-rpath,{LIB}:{oracle_dir}:{os.path.join(CUDA_HOME, 'lib64')}"])
    return out


def build_all(force: bool = False) -> None:
    if shutil.which(NVCC) is None and not os.path.exists(NVCC):
        raise RuntimeError(f"nvcc not found at {NVCC}")
    build_cuda(force)
    build_oracle(force)
    build_host(force)
    build_bindings(force)
    build_tests(force)
    build_gpu_tests(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
