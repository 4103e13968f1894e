"""Multi-rank parity check, one process per GPU (launched by torchrun from
tests/test_multigpu.py or by hand):

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29511 tests/mp_round_check.py --wire fp16

Every rank hosts `--peers-per-rank` peers; the round runs over CUDA IPC /
NVLink between the ranks. Every rank checks its own all-gathered averaged
vector and its LAMB replica against the CPU oracle of the whole G-peer round
(bit-exact given the device trust ratios) and that all replicas agree.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402
from paper_2106_10207_b200 import AveragingRound, fill_synthetic  # noqa: E402
from paper_2106_10207_b200 import _native as nat  # noqa: E402

HP = dict(lr=1.76e-3, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.01, bias_correction=1)
SIGMA = float(np.float32(1e-3 * np.sqrt(3.0)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--wire", default="fp16")
    ap.add_argument("--peers-per-rank", type=int, default=1)
    ap.add_argument("--fractions", default="")
    ap.add_argument("--weights", default="")
    ap.add_argument("--sizes", default="3,1000,70001,2,4096,131075,5")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--block", type=int, default=4096)
    ap.add_argument("--shard-lamb", action="store_true",
                    help="sharded LAMB: owners step their range, parameters pushed to all ranks")
    ap.add_argument("--accumulate", action="store_true",
                    help="device-side accumulation: per-peer micro-batches, sample-count weights")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = args.peers_per_rank
    G = L * world
    sizes = [int(x) for x in args.sizes.split(",")]
    n = sum(sizes)
    fr = [float(x) for x in args.fractions.split(",")] if args.fractions else [1.0 / G] * G
    w = [float(x) for x in args.weights.split(",")] if args.weights else [float(g + 1) for g in range(G)]
    assert len(fr) == G and len(w) == G
    wire, block = args.wire, args.block

    rnd = AveragingRound(n, sizes, wire=wire, q8_block=block, peers_per_rank=L, rank=rank,
                         world=world, device=local, lr=HP["lr"], eps=HP["eps"],
                         weight_decay=HP["weight_decay"], barrier_timeout_s=30.0,
                         shard_lamb=args.shard_lamb)
    rnd.assign(fr, w)
    lo, hi = rnd.own_range() if args.shard_lamb else (0, n)
    grads = []
    for l in range(L):
        g = rank * L + l
        if w[g] == 0:
            grads.append(None)
            continue
        t = torch.empty(n, device="cuda")
        fill_synthetic(t, 21, g, SIGMA)
        grads.append(t)
    p = rnd.param_buffer() if args.shard_lamb else torch.empty(n, device="cuda")
    fill_synthetic(p, 22, 0, 0.02, 0)
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")

    # oracle state (every rank computes it; cheap at this size)
    grads_h = [None if w[g] == 0 else O.fill_synthetic(n, 21, g, SIGMA) for g in range(G)]
    packed = [None if x is None else O.pack(wire, x, block) for x in grads_h]
    ph = O.fill_synthetic(n, 22, 0, 0.02, 0)
    mh = np.zeros(n, np.float32)
    vh = np.zeros(n, np.float32)
    wires = [np.zeros(1, np.float32) if q is None else q[0] for q in packed]
    scales = [None if q is None else q[1] for q in packed]
    avg, avg_s = O.reduce(wire, wires, scales, w, 0, n, n, block)

    if args.accumulate:  # peer g accumulates g % 3 + 1 micro-batches of g + 1 samples each
        micro = {g: [(k, float(g + 1)) for k in range(g % 3 + 1)] for g in range(G)}
        grads_h = []
        w = []
        for g in range(G):
            acc = None
            for k, _ in micro[g]:
                x = O.fill_synthetic(n, 31 + k, g, SIGMA)
                acc = x.copy() if acc is None else (acc + x).astype(np.float32)
            grads_h.append(acc)
            w.append(sum(s for _, s in micro[g]))
        packed = [O.pack(wire, x, block) for x in grads_h]
        wires = [q[0] for q in packed]
        scales = [q[1] for q in packed]
        avg, avg_s = O.reduce(wire, wires, scales, w, 0, n, n, block)

    errors = []
    for step in range(1, args.steps + 1):
        if args.accumulate:
            buf = step % 2
            for l in range(L):
                g = rank * L + l
                for k, smp in micro[g]:
                    t = torch.empty(n, device="cuda")
                    fill_synthetic(t, 31 + k, g, SIGMA)
                    rnd.accumulate(l, t, smp, buf=buf)
            rnd.run_accumulated(p, m, v, step, buf=buf)
        else:
            rnd.run(grads, p, m, v, step)
        torch.cuda.synchronize()
        got, gs = rnd.read_wire(nat.SP_BUF_AVG)
        have = np.zeros(n, bool)  # sharded: the average stays with the owner
        if not args.shard_lamb:
            have[:] = True
        have[lo:hi] = True
        if not np.array_equal(got[have], avg[have]):
            errors.append(f"step {step}: averaged vector differs ({int((got != avg).sum())} elems)")
        if wire == "q8":
            hs = np.zeros(len(avg_s), bool)
            if not args.shard_lamb:
                hs[:] = True
            hs[lo // block:(hi + block - 1) // block] = True
        if wire == "q8" and not np.array_equal(gs[hs], avg_s[hs]):
            errors.append(f"step {step}: averaged q8 scales differ")
        trust = rnd.read_trust()
        O.lamb(wire, avg, avg_s, ph, mh, vh, sizes, HP, step, block, trust_in=trust)
        # sharded: m and v are kept on the owned range only; p everywhere
        keep = np.zeros(n, bool)
        if not args.shard_lamb:
            keep[:] = True
        keep[lo:hi] = True
        for name, dev, host, msk in (("m", m, mh, keep), ("v", v, vh, keep), ("p", p, ph, None)):
            d = dev.cpu().numpy()
            if not (np.array_equal(d, host) if msk is None else np.array_equal(d[msk], host[msk])):
                errors.append(f"step {step}: {name} differs")
    # all replicas identical
    digest = torch.tensor([float(p.double().sum()),
                           0.0 if args.shard_lamb else float(m.double().sum())], device="cuda")
    allg = [torch.zeros_like(digest) for _ in range(world)]
    dist.all_gather(allg, digest)
    if any(not torch.equal(allg[0], x) for x in allg):
        errors.append("replicas disagree across ranks")
    t = {} if args.accumulate else rnd.run_phased(grads, p, m, v, args.steps + 1)
    res = {"rank": rank, "world": world, "G": G, "wire": wire, "errors": errors, "phases": t}
    out = [None] * world
    dist.all_gather_object(out, res)
    rnd.close()
    if rank == 0:
        print(json.dumps({"ok": all(not r["errors"] for r in out), "ranks": out}))
    dist.barrier()
    dist.destroy_process_group()
    return 0 if all(not r["errors"] for r in out) else 1


if __name__ == "__main__":
    sys.exit(main())
