"""Recipe for oracle/_ref: the reference's OWN code, compiled from its sources
where they lie under /root/reference (never copied into this repo).

    python oracle/build_ref.py [--force]

Builds oracle/_ref/libswarmplan_ref.so from
  /root/reference/proj/src/groups.cpp   build_plan, run_plan (the averaging)
  /root/reference/proj/src/model.cpp    validate, spec_from_json, spec_to_json,
                                        assignment_to_json
  oracle/ref_wrap.cpp                   our extern "C" entry points
with two include shims (oracle/ref_shim/): <Eigen/Dense> -> the dense subset
in include/swarmplan/eigen_compat.hpp (Eigen is not installed) and <json.hpp>
-> the image's nlohmann json 3.11.3. The rest of the reference cannot be
built here: lp.cpp needs SuiteSparse KLU and Eigen/SparseCore, strategy.cpp
and netsim.cpp need lp.cpp, auth.cpp needs libsodium.

TEST INFRASTRUCTURE ONLY (tests/, bench.py's reference arm). Every symbol but
the ref_* entry points is hidden, so the reference's swarmplan:: functions
never interpose on the product's. oracle/_ref/ is git-ignored and travels to
the GPU box with the snapshot (the box has no /root/reference).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = "/root/reference/proj"
OUT = os.path.join(HERE, "_ref", "libswarmplan_ref.so")
SOURCES = [os.path.join(REF, "src", "groups.cpp"), os.path.join(REF, "src", "model.cpp")]
WRAP = os.path.join(HERE, "ref_wrap.cpp")


def _json_include() -> str:
    for cand in glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "include",
                                       "cudnn_frontend", "thirdparty")) + ["/usr/include"]:
        if os.path.exists(os.path.join(cand, "nlohmann", "json.hpp")):
            return cand
    raise RuntimeError("nlohmann/json.hpp not found")


def available() -> bool:
    return all(os.path.exists(s) for s in SOURCES)


def build(force: bool = False) -> str | None:
    """Compiles the library when /root/reference is present; returns its path
    (or None when neither the sources nor a prebuilt library exist)."""
    if not available():
        return OUT if os.path.exists(OUT) else None
    deps = SOURCES + [WRAP] + glob.glob(os.path.join(HERE, "ref_shim", "**", "*"), recursive=True)
    deps += [os.path.join(ROOT, "include", "swarmplan", "eigen_compat.hpp")]
    if not force and os.path.exists(OUT) and all(os.path.getmtime(d) <= os.path.getmtime(OUT)
                                                  for d in deps if os.path.isfile(d)):
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = ["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-fvisibility=hidden",
           "-fvisibility-inlines-hidden", "-Wl,-Bsymbolic", "-ffp-contract=off",
           # the reference's headers first, so "swarmplan/*.hpp" are ITS headers
           f"-I{os.path.join(REF, 'include')}", f"-I{os.path.join(HERE, 'ref_shim')}",
           f"-I{_json_include()}", "-o", OUT, *SOURCES, WRAP, "-pthread"]
    print("[build]", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
