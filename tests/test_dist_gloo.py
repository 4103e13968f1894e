"""Multi-rank host logic on CPU (torch.distributed gloo, world size 2): the
IPC-handle all-gather, plan agreement across ranks and rank ranges. The
GPU data path itself is covered by tests/test_multigpu.py."""
import json
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec_json, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2106_10207_b200 import dist as D

    try:
        blob = D.exchange_handles(bytes([rank]) * 64)
        plan = D.plan_round(spec_json, 17847474, 8)
        D.check_same_plan(plan["offsets"], plan["weights"])
        lo, hi = D.rank_range(plan["offsets"], rank, 4)
        bad = None
        try:  # a rank with a different plan must be refused on every rank
            D.check_same_plan(plan["offsets"], [w + rank for w in plan["weights"]])
        except RuntimeError as e:
            bad = str(e)
        q.put((rank, blob, plan["offsets"], lo, hi, bad))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_logic():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden.fleets import spec_json

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    sj = spec_json("het8c")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, sj, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, b0, o0, lo0, hi0, bad0), (r1, b1, o1, lo1, hi1, bad1) = res
    assert b0 == b1 == bytes([0]) * 64 + bytes([1]) * 64  # rank order
    assert o0 == o1  # deterministic LP: identical plans on every rank
    assert (lo0, hi1) == (0, 17847474) and hi0 == lo1  # 2 ranks x 4 peers tile the vector
    assert bad0 and bad1 and "disagree" in bad0
