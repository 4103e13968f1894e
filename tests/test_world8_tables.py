"""The exchange pointer tables at world sizes no box here has (8 ranks),
host-only: sp_round_describe runs the same pack_plan / push-order code the
executor enqueues with, without touching a device. Checked for every rank
of 8 (and 2 x 4 with virtual peers): the scatter visits every nonempty owner
range exactly once starting with the next rank, covers the whole vector in
wire units, gives each range at least one CTA, and every push to all ranks
ends with the rank itself."""
import ctypes
import json

import pytest

from paper_2106_10207_b200 import _native as nat
from paper_2106_10207_b200 import fleets
from paper_2106_10207_b200.dist import plan_round

N = 17847474
SIZES = json.load(open(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                                  "tensor_tables.json")))["albert-large"]


def _cfg(rank, world, L, wire, shard=False):
    sizes = (ctypes.c_int64 * len(SIZES))(*SIZES)
    c = nat.SpRoundCfg(device=0, rank=rank, world=world, peers_per_rank=L, n=N,
                       wire=nat.WIRE_FORMATS[wire], q8_block=4096, num_tensors=len(SIZES),
                       tensor_sizes=sizes, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.01,
                       bias_correction=1, barrier_timeout_s=20.0, shard_lamb=int(shard))
    return c, sizes


def _describe(rank, world, L, wire, offsets, shard=False):
    c, keep = _cfg(rank, world, L, wire, shard)
    off = (ctypes.c_int64 * len(offsets))(*offsets)
    d = nat.SpPlanDesc()
    nat.check(nat.lib().sp_round_describe(ctypes.byref(c), off, 148, ctypes.byref(d)))
    return d


def _plans():
    out = []
    for wire, align in (("fp16", 8), ("q8", 4096), ("fp32", 8)):
        out.append(("uniform8", wire, 1, plan_round(json.dumps(fleets.homogeneous(8, 1.0, 1000.0, 4096.0, N)),
                                                   N, align)["offsets"]))
        out.append(("het8c", wire, 1, plan_round(fleets.spec_json("het8c"), N, align)["offsets"]))
        out.append(("het8c-2x4", wire, 2, plan_round(fleets.spec_json("het8c"), N, align)["offsets"]))
    return out


@pytest.mark.parametrize("name,wire,L,offsets", _plans(), ids=lambda x: x if isinstance(x, str) else "")
def test_world8_pack_and_push_tables(name, wire, L, offsets):
    G = len(offsets) - 1
    world = G // L
    for rank in range(world):
        d = _describe(rank, world, L, wire, offsets)
        unit = d.unit_elems
        owners = [d.pack_owner[j] for j in range(d.pack_ranges)]
        nonempty = [k for k in range(world) if offsets[(k + 1) * L] > offsets[k * L]]
        # every nonempty owner once, visited from the next rank on
        assert sorted(owners) == nonempty
        order = [(rank + s) % world for s in range(1, world + 1)]
        assert owners == [k for k in order if k in nonempty]
        # ranges in wire units cover each owner's elements
        for j, k in enumerate(owners):
            lo, hi = offsets[k * L], offsets[(k + 1) * L]
            assert d.pack_first_unit[j] == lo // unit
            assert d.pack_units[j] == -(-hi // unit) - lo // unit
            assert d.pack_cta_begin[j + 1] - d.pack_cta_begin[j] >= 1
        assert d.pack_cta_begin[0] == 0 and d.pack_cta_begin[d.pack_ranges] == d.pack_ctas
        assert d.pack_ctas <= 148 * 16
        # K2 range and the push order (self last, every rank once)
        assert (d.own_lo, d.own_hi) == (offsets[rank * L], offsets[(rank + 1) * L])
        push = [d.push_order[k] for k in range(world)]
        assert push[-1] == rank and sorted(push) == list(range(world))
        assert push[0] == (rank + 1) % world
        assert d.avg_push_ranks == world
    # the rotation spreads the first targets: every rank starts with a different owner
    firsts = [_describe(r, world, L, wire, offsets).pack_owner[0] for r in range(world)]
    if all(offsets[(k + 1) * L] > offsets[k * L] for k in range(world)):
        assert sorted(firsts) == list(range(world))


def test_world8_sharded_keeps_the_average_local():
    offsets = plan_round(json.dumps(fleets.homogeneous(8, 1.0, 1000.0, 4096.0, N)), N, 8)["offsets"]
    d = _describe(3, 8, 1, "fp16", offsets, shard=True)
    assert d.avg_push_ranks == 1


def test_describe_rejects_bad_offsets():
    c, keep = _cfg(0, 8, 1, "fp16")
    off = (ctypes.c_int64 * 9)(*([0] * 8 + [N - 1]))
    d = nat.SpPlanDesc()
    assert nat.lib().sp_round_describe(ctypes.byref(c), off, 148, ctypes.byref(d)) == nat.SP_ERR_ARG
