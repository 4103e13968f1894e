"""World size 8 (the driver's 8-GPU scaling run) on whatever GPUs the box has.

tests/test_multigpu.py runs one process per GPU, so on a 1- to 4-GPU box it
never reaches world 8. Here 8 ranks share the visible GPUs (rank r on GPU
r % count, gloo plumbing) and run the same CUDA IPC round: pointer tables,
flag arrays, rotated traversal and push orders, owner ranges and the sharded
LAMB norm exchange all see world = 8. Ranks on one GPU time-slice, so this
checks parity only, never speed.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))
SIZES = "3,1000,70001,2,4096,33000,5"


def _launch(nproc, *extra):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(HERE, "mp_round_check.py"), "--oversubscribe", "--sizes", SIZES,
           "--steps", "2", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=420)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"], res
    assert res["ranks"][0]["world"] == nproc
    return res


@pytest.mark.parametrize("wire", ["fp16", "q8"])
def test_world8_replicated(wire):
    _launch(8, "--wire", wire)


def test_world8_sharded_lamb_nonuniform_with_client():
    # het8c-like split: six 1/20 parts, a client with nothing, a 7/10 owner
    fr = ",".join(["0.05"] * 6 + ["0", "0.7"])
    _launch(8, "--wire", "fp16", "--shard-lamb", "--fractions", fr)
