"""Compile-time configurations of k_lamb for A/B runs on the GPU box
(scripts/gpu/variants.sh): build/variants/<name>/libsp_round.so.

    python scripts/build_variants.py w16c1s3 w8c2s3 trace

<name> = w<warps>c<CTAs per SM>s<stages>[v<float4 per thread>], or "trace" (the default
configuration with SP_LAMB_TRACE, for scripts/micro/lamb_trace.py).
"""
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2106_10207_b200", "csrc", "cuda", "sp_round.cu")


def flags(name):
    if name == "trace":
        return ["-DSP_LAMB_TRACE"]
    m = re.fullmatch(r"w(\d+)c(\d+)s(\d+)(?:v(\d+))?", name)
    if not m:
        raise SystemExit(f"bad variant {name}")
    out = [f"-DSP_LAMB_WARPS={m.group(1)}", f"-DSP_LAMB_CTAS={m.group(2)}", f"-DSP_LAMB_STAGES={m.group(3)}"]
    if m.group(4):
        out.append(f"-DSP_LAMB_VEC={m.group(4)}")
    return out


def build(name):
    d = os.path.join(ROOT, "build", "variants", name)
    os.makedirs(d, exist_ok=True)
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", f"-I{os.path.join(ROOT, 'include')}", *flags(name),
           "-Xptxas", "-v", "-o", os.path.join(d, "libsp_round.so"), SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    lines = r.stderr.splitlines()
    i = next(k for k, x in enumerate(lines) if "k_lamb" in x and "Compiling" in x)
    stats = [x.split(":", 1)[-1].strip() for x in lines[i + 1:i + 4] if "spill" in x or "registers" in x]
    return f"{name}: {' | '.join(stats)}"


if __name__ == "__main__":
    with ThreadPoolExecutor(8) as ex:
        for line in ex.map(build, sys.argv[1:]):
            print(line)
