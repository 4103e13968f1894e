"""Per-CTA timeline of one k_lamb launch (SP_LAMB_TRACE build): where the
time goes: when each CTA ran out of pass-1 chunks, left the stream loop and exited.

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
    S = 64 + 128 * 8  # sp_lamb.cuh kLambTraceStride
    buf = np.zeros(148 * 8 * S, np.uint64)
    grid = lib.sp_round_lamb_trace(r._h, buf.ctypes.data, buf.size)
    tr = buf[: grid * S].reshape(grid, S).astype(np.int64)
    t = tr[:, :64]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3  # us
    span = rel[:, 3].max()
    print(f"grid {grid}, chunks {r.lamb_chunks()[0]}, kernel span {span:.1f} us "
          f"(start spread {rel[:, 0].max():.2f} us)")
    for k, name in ((1, "pass-1 counts done"), (2, "stream loop done"), (3, "exit")):
        x = rel[:, k]
        print(f"{name:20s} min/med/max {x.min():7.1f} {np.median(x):7.1f} {x.max():7.1f}")
    print(f"chunks not stashed: {int(t[:, 4].sum())} (max per CTA {int(t[:, 4].max())})")
    print(f"tail after the last pass-1 count: {span - rel[:, 1].max():.1f} us")
    drain0 = (t[:, 7] - t0) / 1e3
    print(f"first iteration without a pass-1 chunk: min/med/max {drain0.min():.1f} {np.median(drain0):.1f} "
          f"{drain0.max():.1f} us; per CTA: empty iterations median {np.median(t[:, 5]):.0f} "
          f"(max {t[:, 5].max()}), pass-2-only iterations median {np.median(t[:, 6]):.0f} (max {t[:, 6].max()})")
    # per-iteration phases (SM clocks): data warp 0: 0 top, 1 slot and stage
    # ready, 2 pass 1 done, 3 pass 2 done, 4 reported done; claims lane: 5
    # iteration reported done by every data warp, 6 next slot filled, 7 armed
    it = tr[:, 64:].reshape(grid, 128, 8).astype(np.float64)
    ok = (it[:, :-1, 0] > 0) & (it[:, 1:, 0] > 0)
    d = lambda a, b: (it[:, :-1, b] - it[:, :-1, a])[ok]
    per = (it[:, 1:, 0] - it[:, :-1, 0])[ok]
    print(f"iterations traced: {int(ok.sum())}; cycles per iteration median {np.median(per):.0f}")
    for (a, b, name) in ((0, 1, "wait for slot+stage"), (1, 2, "pass 1"), (2, 3, "pass 2"),
                         (3, 4, "reduce + report"), (4, 5, "last warp -> claims"), (5, 6, "claims: fill+pick"),
                         (6, 7, "claims: arm")):
        x = d(a, b)
        print(f"  {name:22s} median {np.median(x):8.0f}  mean {x.mean():8.0f}  p90 {np.percentile(x, 90):8.0f}")

    r.close()


if __name__ == "__main__":
    main()
