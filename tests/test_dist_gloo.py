"""Multi-rank host logic on CPU (torch.distributed gloo, world sizes 2 and 8):
the IPC-handle all-gather, plan agreement across ranks and rank ranges. World
8 is the driver's 8-GPU scaling run, which no test box here reaches (the
GPU data path is covered up to 4 GPUs by tests/test_multigpu.py; ranks that
spin on each other must never share a GPU)."""
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


def _worker(rank, world, port, spec_json, q, L):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2106_10207_b200 import dist as D

    try:
        blob = D.exchange_handles(bytes([rank]) * 64)
        plan = D.plan_round(spec_json, 17847474, 8)
        D.check_same_plan(plan["offsets"], plan["weights"])
        lo, hi = D.rank_range(plan["offsets"], rank, L)
        bad = None
        try:  # a rank with a different plan must be refused on every rank
            D.check_same_plan(plan["offsets"], [w + rank for w in plan["weights"]])
        except RuntimeError as e:
            bad = str(e)
        q.put((rank, blob, plan["offsets"], lo, hi, bad))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_gloo_host_logic(world):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden.fleets import FRACTIONS_APPENDIX_A, spec_json

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    sj = spec_json("het8c")  # 8 peers: L = 8 / world per rank
    L = 8 // world
    procs = [ctx.Process(target=_worker, args=(r, world, port, sj, q, L)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_blob = b"".join(bytes([r]) * 64 for r in range(world))
    for r, (rank, blob, offs, lo, hi, bad) in enumerate(res):
        assert rank == r
        assert blob == want_blob  # rank order
        assert offs == res[0][2]  # deterministic LP: identical plans on every rank
        assert bad and "disagree" in bad  # a rank with a different plan is refused everywhere
        assert (lo, hi) == (offs[r * L], offs[(r + 1) * L])
    # ranks tile the vector: contiguous, first at 0, last at n
    assert res[0][3] == 0 and res[-1][4] == 17847474
    assert all(res[k][4] == res[k + 1][3] for k in range(world - 1))
    if world == 8:  # het8c: 1/20 x6, a client with nothing, 7/10
        sizes = [hi - lo for (_, _, _, lo, hi, _) in res]
        want = [f * 17847474 for f in FRACTIONS_APPENDIX_A["het8c"]]
        assert sizes[6] == 0
        assert all(abs(s - w) <= 8 for s, w in zip(sizes, want))


def _fd_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2106_10207_b200 import dist as D

    try:
        fd = None
        if rank == 1:  # the source need not be rank 0
            fd = os.memfd_create("sp-test")
            os.write(fd, b"multicast handle stand-in")
        got = D.share_fd(fd, src=1)
        q.put((rank, os.pread(got, 64, 0)))
        os.close(got)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_share_fd_between_ranks(world):
    # the POSIX-fd path CUDA multicast / VMM handles need between processes
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_fd_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r for r, _ in res] == list(range(world))
    assert all(b == b"multicast handle stand-in" for _, b in res)
