"""Multi-rank host plumbing of the round (one process per GPU).

torch.distributed is used only to move a few bytes between processes: the
CUDA IPC handle blobs of every rank (sp_round_export / sp_round_connect) and
the sanity check that every rank planned the same assignment. The data path
itself never touches torch.distributed (NVLink stores from the kernels).
"""
from __future__ import annotations

import hashlib
import json


def exchange_handles(blob: bytes, group=None) -> bytes:
    """All-gather one opaque blob per rank; returns the concatenation in rank
    order (what sp_round_connect expects)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out: list = [None] * world
    dist.all_gather_object(out, bytes(blob), group=group)
    sizes = {len(b) for b in out}
    if len(sizes) != 1:
        raise RuntimeError(f"ranks exported handle blobs of different sizes: {sorted(sizes)}")
    return b"".join(out)


def plan_round(spec_json: str, n: int, align: int, sample_counts=None) -> dict:
    """LP plan shared by every rank: fractions from solve_strategy, part
    offsets, weights (sample counts; default samples_per_sec * duty cycle,
    the accumulation the LP assumed, /root/reference/proj/src/netsim.cpp:158)."""
    from . import _swarmplan

    plan = _swarmplan.plan_parts(spec_json, n, align)
    if sample_counts is None:
        spec = json.loads(spec_json)
        sample_counts = [p.get("samples_per_sec", 0.0) * c
                         for p, c in zip(spec["peers"], plan["duty_cycle"])]
    plan["weights"] = [float(w) for w in sample_counts]
    return plan


def rank_range(offsets, rank: int, peers_per_rank: int) -> tuple[int, int]:
    """Element range rank `rank` owns: the union of its peers' parts."""
    return int(offsets[rank * peers_per_rank]), int(offsets[(rank + 1) * peers_per_rank])


def plan_digest(offsets, weights) -> str:
    h = hashlib.sha256()
    h.update(json.dumps([list(map(int, offsets)), list(map(float, weights))]).encode())
    return h.hexdigest()


def check_same_plan(offsets, weights, group=None) -> None:
    """Every rank must run the round with the same offsets and weights (a
    mismatch would make owners disagree about who reduces what)."""
    import torch.distributed as dist

    mine = plan_digest(offsets, weights)
    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, mine, group=group)
    if any(d != mine for d in out):
        raise RuntimeError("ranks disagree on the round assignment (offsets/weights)")


def share_fd(fd: int | None, src: int = 0, group=None, tag: str = "sp", timeout_s: float = 60.0) -> int:
    """Give every rank of one node a file descriptor owned by rank `src`.

    CUDA multicast objects and VMM allocations are shared between processes
    as POSIX file descriptors (cuMemExportToShareableHandle), which cannot
    travel through torch.distributed. Rank `src` listens on an abstract Unix
    socket whose name (with a random nonce) it all-gathers together with
    every rank's pid; every other rank connects and receives the descriptor
    with SCM_RIGHTS. The source hands the descriptor only to a peer whose
    SO_PEERCRED pid and uid are one of the job's ranks (a descriptor maps GPU
    memory of the job), each once, and gives up after `timeout_s`. Returns
    the local descriptor (`fd` itself on `src`; the caller closes received
    ones)."""
    import os
    import secrets
    import socket
    import struct

    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    info: list = [None] * world
    name = f"\0{tag}-{secrets.token_hex(16)}" if rank == src else None
    dist.all_gather_object(info, (name, os.getpid(), os.getuid()), group=group)
    path = info[src][0]
    if rank == src:
        if fd is None:
            raise ValueError("the source rank must pass a descriptor")
        expected = {(pid, uid) for r, (_, pid, uid) in enumerate(info) if r != src}
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(path)
        srv.listen(world)
        srv.settimeout(timeout_s)
        dist.barrier(group=group)  # listening before anyone connects
        try:
            while expected:
                conn, _ = srv.accept()
                with conn:
                    cred = conn.getsockopt(socket.SOL_SOCKET, socket.SO_PEERCRED, struct.calcsize("3i"))
                    pid, uid, _ = struct.unpack("3i", cred)
                    if (pid, uid) not in expected:
                        continue  # not one of this job's ranks (or already served)
                    expected.discard((pid, uid))
                    socket.send_fds(conn, [b"fd"], [fd])
        finally:
            srv.close()
        dist.barrier(group=group)
        return fd
    dist.barrier(group=group)
    with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as c:
        c.settimeout(timeout_s)
        c.connect(path)
        _, fds, _, _ = socket.recv_fds(c, 16, 1)
    dist.barrier(group=group)
    if len(fds) != 1:
        raise RuntimeError("share_fd: no descriptor received")
    return fds[0]
