"""Per-CTA timeline of one k_lamb launch (SP_LAMB_TRACE build): where the
time goes between pass 1, the split-phase window barriers and pass 2.

    python scripts/micro/lamb_trace.py path/to/traced/libsp_round.so [workload]
"""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2106_10207_b200 import _native as nat
    nat.LIB_PATH = sys.argv[1]
    from paper_2106_10207_b200 import AveragingRound, fill_synthetic

    table = sys.argv[2] if len(sys.argv) > 2 else "albert-large"
    wire = sys.argv[3] if len(sys.argv) > 3 else "fp16"
    sizes = json.load(open(os.path.join(ROOT, "tests", "golden", "tensor_tables.json")))[table]
    n = sum(sizes)
    g = torch.empty(n, device="cuda")
    fill_synthetic(g, 1, 0, 1e-3)
    p = torch.empty(n, device="cuda")
    fill_synthetic(p, 2, 0, 0.02, 0)
    m, v = torch.zeros_like(p), torch.zeros_like(p)
    r = AveragingRound(n, sizes, wire=wire)
    r.assign([1.0], [1.0])
    for step in range(1, 21):
        r.run([g], p, m, v, step)
    torch.cuda.synchronize()
    lib = nat.lib()
    lib.sp_round_lamb_trace.restype = ctypes.c_int
    lib.sp_round_lamb_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    buf = np.zeros(148 * 8 * 64, np.uint64)
    grid = lib.sp_round_lamb_trace(r._h, buf.ctypes.data, buf.size)
    t = buf[: grid * 64].reshape(grid, 64).astype(np.int64)
    W = r.lamb_windows()
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3  # us
    print(f"grid {grid}, windows {W}, kernel span {rel[:, 3 * W].max():.1f} us "
          f"(start spread {rel[:, 0].max():.2f} us)")
    for w in range(W):
        p1 = rel[:, 1 + 3 * w]
        wt = rel[:, 2 + 3 * w]
        p2 = rel[:, 3 + 3 * w]
        prev = rel[:, 0] if w == 0 else np.maximum(rel[:, 3 * w], rel[:, 1 + 3 * (w - 1)] * 0)
        print(f"w{w}: pass1 end min/med/max {p1.min():7.1f} {np.median(p1):7.1f} {p1.max():7.1f} | "
              f"wait end {wt.min():7.1f} {np.median(wt):7.1f} {wt.max():7.1f} | "
              f"pass2 end {p2.min():7.1f} {np.median(p2):7.1f} {p2.max():7.1f}")
    # time each CTA spends waiting at window barriers
    waits = np.zeros(grid)
    for w in range(W):
        before = rel[:, 1 + 3 * (w + 1)] if w + 1 < W else rel[:, 1 + 3 * w]
        waits += np.maximum(0, rel[:, 2 + 3 * w] - before)
    print(f"barrier wait per CTA: median {np.median(waits):.1f} us, max {waits.max():.1f} us")
    sm = np.arange(grid) % 148
    per_sm = [rel[sm == k, 1].max() for k in range(148)]
    print(f"window-0 pass-1 end by SM: min {min(per_sm):.1f} max {max(per_sm):.1f}")
    r.close()


if __name__ == "__main__":
    main()
