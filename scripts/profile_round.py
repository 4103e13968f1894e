"""Small fixed workload for ncu: W warm-up + K rounds of the ALBERT-large
fp16 round on one GPU (G = --peers virtual peers), no timing soak."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2106_10207_b200 import AveragingRound, fill_synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--wire", default="fp16")
ap.add_argument("--table", default="albert-large")
ap.add_argument("--peers", type=int, default=1)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--phased", action="store_true")
a = ap.parse_args()
sizes = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                                    "tensor_tables.json")))[a.table]
n = sum(sizes)
grads = []
for g in range(a.peers):
    t = torch.empty(n, device="cuda")
    fill_synthetic(t, 1, g, 1.7e-3)
    grads.append(t)
p = torch.empty(n, device="cuda")
fill_synthetic(p, 2, 0, 0.02, 0)
m = torch.zeros(n, device="cuda")
v = torch.zeros(n, device="cuda")
r = AveragingRound(n, sizes, wire=a.wire, peers_per_rank=a.peers)
r.assign([1.0 / a.peers] * a.peers, [1.0] * a.peers)
for s in range(1, a.steps + 1):
    if a.phased:
        print(r.run_phased(grads, p, m, v, s))
    else:
        r.run(grads, p, m, v, s)
torch.cuda.synchronize()
print("ok")
