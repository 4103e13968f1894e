"""Multi-GPU round (one process per GPU over CUDA IPC / NVLink) vs the oracle.

Launches tests/mp_round_check.py under torchrun on every visible GPU (2..8);
skipped on a single-GPU box (the same kernels and pointer tables are
exercised with virtual peers by tests/test_round_gpu.py).
"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

torch = pytest.importorskip("torch")
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
if NGPU < 2:
    pytest.skip("needs >= 2 GPUs", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _launch(nproc, *extra, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(HERE, "mp_round_check.py"), *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env=None if env is None else {**os.environ, **env})
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"], res
    return res


@pytest.mark.parametrize("wire", ["fp32", "fp16", "q8"])
def test_uniform_all_gpus(wire):
    _launch(NGPU, "--wire", wire)


def test_nonuniform_with_client_and_virtual_peers():
    # 2 peers per GPU; one zero-length part (client) and one zero-weight peer
    G = 2 * NGPU
    fr = [0.0] + [1.0 / (G - 1)] * (G - 1)
    w = [3.0] * G
    w[G - 1] = 0.0
    _launch(NGPU, "--wire", "fp16", "--peers-per-rank", "2", "--fractions",
            ",".join(map(str, fr)), "--weights", ",".join(map(str, w)))


def test_owner_takes_everything_q8():
    # aux_server-like: one GPU aggregates 100% (test_strategy.cpp:197-207)
    fr = [0.0] * NGPU
    fr[-1] = 1.0
    _launch(NGPU, "--wire", "q8", "--fractions", ",".join(map(str, fr)))


@pytest.mark.parametrize("wire", ["fp16", "q8"])
def test_device_accumulation_multi_gpu(wire):
    """Micro-batches accumulated on each GPU; sample counts published over
    NVLink weight the average; buffers alternate per step (DPU)."""
    _launch(NGPU, "--wire", wire, "--peers-per-rank", "2", "--accumulate")


@pytest.mark.parametrize("wire", ["fp32", "fp16", "q8"])
def test_sharded_lamb(wire):
    """ZeRO-1 style LAMB: owners step their range; per-tensor
    norms cross NVLink; parameters pushed to every rank. p bit-exact on every
    rank given the device trust; m, v bit-exact on the owned range."""
    _launch(NGPU, "--wire", wire, "--shard-lamb")


def test_sharded_lamb_ragged_owners():
    # a rank that owns nothing (zero-length parts) still publishes zero norms
    # and receives every parameter
    fr = [0.0] * NGPU
    fr[-1] = 0.6
    fr[0] = 0.4
    _launch(NGPU, "--wire", "fp16", "--shard-lamb", "--fractions", ",".join(map(str, fr)))
    _launch(NGPU, "--wire", "q8", "--shard-lamb", "--peers-per-rank", "2", "--accumulate")


def test_sharded_lamb_many_steps_nonuniform():
    # several rounds through the cached graph; the in-kernel norm exchange
    # and the counter resets must hold across replays
    _launch(NGPU, "--wire", "fp16", "--shard-lamb", "--steps", "4")
    fr = [0.0] * NGPU
    fr[-1], fr[0] = 0.7, 0.3
    _launch(NGPU, "--wire", "q8", "--shard-lamb", "--fractions", ",".join(map(str, fr)))
