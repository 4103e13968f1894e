"""Measured executor round times for the reference's strategy comparator
(SURVEY §8f N3). The reference prices an averaging round with a fluid model
(payload / slowest recipient rate, /root/reference/proj/src/netsim.cpp:146-201)
and compare_strategies reports steps/hour from it (:360-382). Here each
algorithm's partition of the fleet is run on the GPU executor and timed, and
those times replace the model's comm time:

  allreduce         uniform parts, 1/G each (strategy.cpp:502-512)
  parameter_server  the best duplex peer owns the whole vector (netsim.cpp:180-195)
  adaptive          the LP load balancer's fractions (strategy.cpp:473-485)

The fleet's G peers are hosted as virtual peers on one GPU (peers_per_rank =
G): the same kernels and pointer tables as G GPUs, with the exchange through
local HBM instead of NVLink. Weights are the peers' sample rates (0 for peers
that do not compute), the sample-count weights of the DeDLOC average.
"""
from __future__ import annotations

import json
from typing import Sequence

from . import _swarmplan
from .round import AveragingRound, fill_synthetic

ALGORITHMS = ("allreduce", "parameter_server", "adaptive")


def _fleet(spec_json: str):
    spec = json.loads(spec_json)
    peers = spec["peers"]
    n = int(round(float(spec["param_count"])))
    w = [float(p.get("samples_per_sec", 0.0)) if p.get("can_compute", True) else 0.0
         for p in peers]
    if not any(x > 0 for x in w):
        w = [1.0] * len(peers)
    return peers, n, w


def _best_duplex(peers) -> int:
    best, bw = 0, -1.0
    for i, p in enumerate(peers):
        d = min(float(p.get("download_mbps", 0.0)), float(p.get("upload_mbps", 0.0)))
        if d > bw:
            best, bw = i, d
    return best


def fractions_for(spec_json: str, algorithm: str) -> list[float]:
    peers, _, _ = _fleet(spec_json)
    G = len(peers)
    if algorithm == "allreduce":
        return [1.0 / G] * G
    if algorithm == "parameter_server":
        f = [0.0] * G
        f[_best_duplex(peers)] = 1.0
        return f
    if algorithm == "adaptive":
        return list(_swarmplan.solve_strategy(spec_json)["fractions"])
    raise ValueError(f"unknown algorithm: {algorithm}")


def measure_round_times(spec_json: str, *, algorithms: Sequence[str] = ALGORITHMS,
                        wire: str = "fp16", tensor_sizes: Sequence[int] | None = None,
                        steps: int = 20, warmup: int = 3, device: int | None = None) -> dict:
    """Seconds per executor round (averaging + LAMB step, CUDA-graph replay,
    median-free mean over `steps` after `warmup`) for each algorithm."""
    import torch

    peers, n, w = _fleet(spec_json)
    G = len(peers)
    dev = torch.cuda.current_device() if device is None else int(device)
    sizes = list(tensor_sizes) if tensor_sizes else [n]
    grads = []
    for g in range(G):
        t = torch.empty(n, device=f"cuda:{dev}")
        fill_synthetic(t, 1, g, 1.7e-3)
        grads.append(t)
    out = {}
    for alg in algorithms:
        rnd = AveragingRound(n, sizes, wire=wire, peers_per_rank=G, device=dev)
        rnd.assign(fractions_for(spec_json, alg), w)
        p = torch.empty(n, device=f"cuda:{dev}")
        fill_synthetic(p, 2, 0, 0.02, 0)
        m = torch.zeros(n, device=f"cuda:{dev}")
        v = torch.zeros(n, device=f"cuda:{dev}")
        st = torch.cuda.Stream(dev)
        with torch.cuda.stream(st):
            step = 0
            for _ in range(max(1, warmup)):
                step += 1
                rnd.run([g if w[i] > 0 else None for i, g in enumerate(grads)], p, m, v, step, st)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(steps):
                step += 1
                rnd.run([g if w[i] > 0 else None for i, g in enumerate(grads)], p, m, v, step, st)
            e1.record(st)
            st.synchronize()
        out[alg] = e0.elapsed_time(e1) / steps / 1e3
        rnd.close()
    return out


def compare_strategies_measured(spec_json: str, **kw) -> list[dict]:
    """compare_strategies with every algorithm's round priced by the executor."""
    measured = measure_round_times(spec_json, **kw)
    rows = _swarmplan.compare_strategies(spec_json, measured)
    for r in rows:
        r["measured_round_s"] = measured.get(r["algorithm"])
    return rows
