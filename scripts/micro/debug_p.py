"""Where pass 2 went wrong: one LAMB step of the albert-large G=8 fp16
parity case; prints the mismatching elements of p grouped by tensor, and
whether they kept their old value (pass 2 skipped) or got another update."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    from oracle import oracle as O
    from paper_2106_10207_b200 import AveragingRound, fill_synthetic
    from paper_2106_10207_b200 import _native as nat
    from test_round_gpu import HP, SIGMA

    sizes = json.load(open(os.path.join(ROOT, "tests", "golden", "tensor_tables.json")))["albert-large"]
    wire, G = sys.argv[1] if len(sys.argv) > 1 else "fp16", int(sys.argv[2]) if len(sys.argv) > 2 else 8
    seed = int(sys.argv[3]) if len(sys.argv) > 3 else 11
    n = sum(sizes)
    weights = [4.0] * G
    grads_h = [O.fill_synthetic(n, seed, g, SIGMA) for g in range(G)]
    p_h = O.fill_synthetic(n, seed + 1, 0, 0.02, 0)
    m_h = np.zeros(n, np.float32)
    v_h = np.zeros(n, np.float32)
    grads_d = []
    for g in range(G):
        t = torch.empty(n, dtype=torch.float32, device="cuda")
        fill_synthetic(t, seed, g, SIGMA)
        grads_d.append(t)
    p_d = torch.from_numpy(p_h.copy()).cuda()
    m_d = torch.zeros(n, device="cuda")
    v_d = torch.zeros(n, device="cuda")
    rnd = AveragingRound(n, sizes, wire=wire, peers_per_rank=G, lr=HP["lr"], betas=(HP["beta1"], HP["beta2"]),
                         eps=HP["eps"], weight_decay=HP["weight_decay"])
    rnd.assign([1 / G] * G, weights)
    packed = [O.pack(wire, x, 4096) for x in grads_h]
    p0 = p_h.copy()
    for step in range(1, 4):
        rnd.run(grads_d, p_d, m_d, v_d, step)
        torch.cuda.synchronize()
        avg, avg_s = O.reduce(wire, [q[0] for q in packed], [q[1] for q in packed], weights, 0, n, n, 4096)
        trust_d = rnd.read_trust()
        before = p_h.copy()
        O.lamb(wire, avg, avg_s, p_h, m_h, v_h, sizes, HP, step, 4096, trust_in=trust_d)
        got = p_d.cpu().numpy()
        bad = np.nonzero(got != p_h)[0]
        print(f"step {step}: m ok {np.array_equal(m_d.cpu().numpy(), m_h)}, {bad.size} p mismatches")
        if bad.size:
            starts = np.cumsum([0] + sizes)
            ts = np.searchsorted(starts, bad, side="right") - 1
            for t in np.unique(ts)[:20]:
                idx = bad[ts == t]
                kept = np.sum(got[idx] == before[idx])
                print(f"  tensor {t} (size {sizes[t]}): {idx.size} bad, {kept} kept the old value, "
                      f"first {idx[:4] - starts[t]}, chunks(2048) {np.unique(idx // 2048)[:8]}")
            p_h = got.copy()  # continue from the device state
    rnd.close()


if __name__ == "__main__":
    main()
