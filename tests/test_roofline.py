"""Byte model and roofline of the round (paper_2106_10207_b200/roofline.py),
the bound bench.py reports and the rule its --lamb auto uses."""
import json

import pytest

from paper_2106_10207_b200 import fleets
from paper_2106_10207_b200.dist import plan_round
from paper_2106_10207_b200.roofline import (choose_shard_lamb, overlap_roofline, rank_model,
                                            round_roofline)

N = 17847474


def _offsets(fleet, G, n=N, align=8):
    sj = fleets.spec_json(fleet) if fleet else json.dumps(fleets.homogeneous(G, 1.0, 1000.0, 4096.0, n))
    return plan_round(sj, n, align)["offsets"]


def test_one_gpu_bytes_match_survey():
    # G = 1 -> pack 4 + b, LAMB 24 + b, no NVLink
    m = rank_model(0, [0, N], 1, 1, N, 2.0, "fp16", False, True)
    assert m["hbm"] == pytest.approx(6.0 + 26.0)
    assert m["nvl"] == 0.0
    # fused pack + LAMB: one launch carries both §8(d) terms (4 + b + 24 + b);
    # the kernel moves 4 + b + 24 + 4 (no wire re-read, p re-read in pass 2)
    assert m["alg"]["lamb_ms"] == pytest.approx(N * 32.0)
    assert m["alg"]["pack_ms"] == 0.0
    assert m["impl"]["lamb_ms"] == pytest.approx(N * 34.0)
    fp32 = rank_model(0, [0, N], 1, 1, N, 4.0, "fp32", False, False)
    assert fp32["hbm"] == pytest.approx(28.0)  # zero-copy wire
    assert fp32["alg"]["lamb_ms"] == pytest.approx(N * 28.0)
    q8 = rank_model(0, [0] + [N] * 8, 8, 1, N, 1.0 + 4 / 4096, "q8", False, False)  # 8 virtual peers
    assert q8["alg"]["pack_ms"] == pytest.approx(8 * N * (5 + 4 / 4096))
    assert q8["alg"]["reduce_ms"] == pytest.approx(9 * N * (1 + 4 / 4096))


def test_uniform_split_bytes():
    offs = _offsets(None, 4)
    m = rank_model(1, offs, 1, 4, N, 2.0, "fp16", True, False)
    assert m["f"] == pytest.approx(0.25, rel=1e-5)  # offsets aligned to 8 elements
    (ph, pn), (rh, rn), (lh, ln) = m["phases"]
    assert pn == pytest.approx(0.75 * 2.0, rel=1e-5)       # scatter out = in
    assert rn == 0.0                                       # sharded: average stays local
    assert ln == pytest.approx(3 * 0.25 * 4.0, rel=1e-5)   # parameter push
    assert lh == pytest.approx(0.25 * 26.0 + 0.75 * 4.0, rel=1e-5)


def test_overlap_bound_is_below_serialized():
    for fleet, G, world in [(None, 4, 4), (None, 8, 8), ("het8c", 8, 4), ("het4b", 4, 2)]:
        offs = _offsets(fleet, G)
        L = G // world
        for shard in (True, False):
            ms = [rank_model(r, offs, L, world, N, 2.0, "fp16", shard, False)
                  for r in range(world)]
            assert overlap_roofline(ms, N, 6524.0) <= round_roofline(ms, N, 6524.0) + 1e-15


def test_auto_lamb_mode():
    assert choose_shard_lamb([0, N], 1, 1, N, 2.0, "fp16") is False  # one GPU: replicated
    for G in (2, 4, 8):  # uniform: sharded (4 B/element pushed, 1/G of the LAMB)
        assert choose_shard_lamb(_offsets(None, G), 1, G, N, 2.0, "fp16") is True
    # het8c on 8 GPUs: the 7/10 owner would push 7 x 0.7 x 4 B per element
    assert choose_shard_lamb(_offsets("het8c", 8), 1, 8, N, 2.0, "fp16") is False


def test_auto_lamb_mode_matches_measured_choices():
    # profiles/r01/lamb_mode.txt (2 and 4 B200s): replicated won every
    # non-uniform fleet, sharded every uniform headline workload
    for fleet, G, world, wire, b in [("het8c", 8, 2, "fp16", 2.0), ("het8c", 8, 4, "fp16", 2.0),
                                     ("het4b", 4, 2, "fp32", 4.0), ("het4b", 4, 4, "fp32", 4.0)]:
        n = 11813810 if fleet == "het4b" else N
        offs = _offsets(fleet, G, n)
        assert choose_shard_lamb(offs, G // world, world, n, b, wire) is False, (fleet, world)
    for world, wire, b in [(2, "fp16", 2.0), (4, "fp16", 2.0), (4, "fp32", 4.0), (4, "q8", 1.0 + 4 / 4096)]:
        offs = _offsets(None, world, N, 4096 if wire == "q8" else 8)
        assert choose_shard_lamb(offs, 1, world, N, b, wire) is True, (world, wire)
