"""Small rounds for compute-sanitizer (memcheck / racecheck / synccheck):
ragged tensor table, 4 virtual peers, every wire format, replicated and
sharded LAMB, a tensor larger than a LAMB window, 2 steps each.

    compute-sanitizer --tool memcheck python scripts/sanitize_round.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2106_10207_b200 import AveragingRound, fill_synthetic  # noqa: E402

for sizes in ([3, 1000, 70001, 2, 4096, 13107, 5], [7, 5_000_001, 9]):
    n = sum(sizes)
    for wire in ("fp32", "fp16", "q8"):
        for shard in (False, True):
            grads = []
            for g in range(4):
                t = torch.empty(n, device="cuda")
                fill_synthetic(t, 3, g, 1e-3)
                grads.append(t)
            r = AveragingRound(n, sizes, wire=wire, peers_per_rank=4, shard_lamb=shard)
            p = r.param_buffer() if shard else torch.empty(n, device="cuda")
            p.fill_(0.02)
            m = torch.zeros(n, device="cuda")
            v = torch.zeros(n, device="cuda")
            r.assign([0.1, 0.2, 0.3, 0.4], [1.0, 2.0, 0.0, 3.0])
            for s in (1, 2):
                r.run_phased(grads, p, m, v, s)
            torch.cuda.synchronize()
            r.close()
print("sanitize round ok")
