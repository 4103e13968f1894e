"""Parity of the CUDA averaging round (through the C-ABI) with the CPU oracle.

Bit-exact: wire codes of every peer (fp16 / q8 codes and scales), the
averaged vector, LAMB moments m and v, and the updated parameters given the
device's trust ratios. Within tolerance: the trust ratios themselves (device
norms are fp32 partial sums, the oracle's are fp64): rtol 2e-5.
Virtual peers (peers_per_rank = G on one GPU) exercise the same kernels and
pointer tables as G GPUs do.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2106_10207_b200 import AveragingRound, fill_synthetic  # noqa: E402
from paper_2106_10207_b200 import _native as nat  # noqa: E402

HP = dict(lr=1.76e-3, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.01, bias_correction=1)
SIGMA = float(np.float32(1e-3 * np.sqrt(3.0)))
HET8C = [1 / 20] * 6 + [0.0, 7 / 10]
HET4B = [1 / 22] * 3 + [19 / 22]
RAGGED = [3, 1000, 70001, 2, 4096, 131075, 5]  # n = 206182, misaligned tensor edges
# p against the oracle's own LAMB: trust ratios agree to rtol 2e-5 and the
# LAMB direction is bounded by |m^|/sqrt(v^) + wd |p| <= ~10 here, so one
# step moves p by at most lr * 10 * 2e-5 more or less than the oracle's
P_ATOL = HP["lr"] * 10 * 2e-5


def _dev(x):
    return torch.from_numpy(x).cuda()


def _run_case(wire, fractions, weights, sizes, steps=1, block=4096, warm=False, seed=11,
              shard=False, offsets=None):
    G = len(fractions)
    n = sum(sizes)
    grads_h = [O.fill_synthetic(n, seed, g, SIGMA) for g in range(G)]
    for g in range(G):
        if weights[g] == 0:
            grads_h[g] = None
    p_h = O.fill_synthetic(n, seed + 1, 0, 0.02, 0)
    m_h = O.fill_synthetic(n, seed + 2, 0, 1e-4, 0) if warm else np.zeros(n, np.float32)
    v_h = np.abs(O.fill_synthetic(n, seed + 3, 0, 1e-6, 0)) if warm else np.zeros(n, np.float32)

    grads_d = []
    for g in range(G):
        if grads_h[g] is None:
            grads_d.append(None)
            continue
        t = torch.empty(n, dtype=torch.float32, device="cuda")
        fill_synthetic(t, seed, g, SIGMA)
        grads_d.append(t)
    p_d, m_d, v_d = _dev(p_h.copy()), _dev(m_h.copy()), _dev(v_h.copy())
    rnd = AveragingRound(n, sizes, wire=wire, q8_block=block, peers_per_rank=G,
                         lr=HP["lr"], betas=(HP["beta1"], HP["beta2"]), eps=HP["eps"],
                         weight_decay=HP["weight_decay"], shard_lamb=shard)
    if shard:  # the round owns the flat parameter vector
        pb = rnd.param_buffer()
        pb.copy_(p_d)
        p_d = pb
    offs = rnd.assign(fractions, weights)
    assert offs[0] == 0 and offs[-1] == n
    if offsets is not None:  # the host LP's plan (C++ part_offsets) == the Python mirror
        assert list(offs) == list(offsets)

    # device synthetic generator == host generator, bit for bit
    for g in range(G):
        if grads_d[g] is not None:
            assert np.array_equal(grads_d[g].cpu().numpy(), grads_h[g])

    packed = [None if x is None else O.pack(wire, x, block) for x in grads_h]
    # the oracle's own LAMB (its fp64 trust ratios) alongside the one fed
    # the device's trust ratios
    p_own, m_own, v_own = p_h.copy(), m_h.copy(), v_h.copy()
    for step in range(1, steps + 1):
        rnd.run(grads_d, p_d, m_d, v_d, step)
        torch.cuda.synchronize()
        # pack: wire codes bit-exact
        for g in range(G):
            if packed[g] is None:
                continue
            got, gs = rnd.read_wire(nat.SP_BUF_WIRE, g)
            np.testing.assert_array_equal(got, packed[g][0], err_msg=f"wire of peer {g}")
            if wire == "q8":
                np.testing.assert_array_equal(gs, packed[g][1])
        # fused reduce-scatter / average / all-gather: bit-exact
        wires = [np.zeros(1, np.float32) if q is None else q[0] for q in packed]
        scales = [None if q is None else q[1] for q in packed]
        avg, avg_s = O.reduce(wire, wires, scales, weights, 0, n, n, block)
        got, gs = rnd.read_wire(nat.SP_BUF_AVG)
        np.testing.assert_array_equal(got, avg, err_msg="averaged vector")
        if wire == "q8":
            np.testing.assert_array_equal(gs, avg_s)
        # LAMB
        trust_d = rnd.read_trust()
        trust_o = O.lamb(wire, avg, avg_s, p_h, m_h, v_h, sizes, HP, step, block, trust_in=trust_d)
        np.testing.assert_allclose(trust_d, trust_o, rtol=2e-5)
        np.testing.assert_array_equal(m_d.cpu().numpy(), m_h, err_msg="m")
        np.testing.assert_array_equal(v_d.cpu().numpy(), v_h, err_msg="v")
        np.testing.assert_array_equal(p_d.cpu().numpy(), p_h, err_msg="p")
        # end to end against the oracle's own trust ratios (P_ATOL per step)
        O.lamb(wire, avg, avg_s, p_own, m_own, v_own, sizes, HP, step, block)
        np.testing.assert_allclose(p_d.cpu().numpy(), p_own, rtol=2e-7, atol=P_ATOL * step,
                                   err_msg="p vs the oracle's own LAMB")
    rnd.close()


@pytest.mark.parametrize("wire", ["fp32", "fp16", "q8"])
@pytest.mark.parametrize("fractions,weights", [
    ([1.0], [32.0]),
    ([0.5, 0.5], [16.0, 16.0]),
    ([1 / 8] * 8, [4.0] * 8),
    (HET8C, [1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0]),
    (HET4B, [3.0, 1.0, 2.0, 7.0]),
])
def test_round_parity_ragged(wire, fractions, weights):
    _run_case(wire, fractions, weights, RAGGED, block=4096 if wire != "q8" else 4096)


@pytest.mark.parametrize("fleet,wire", [("het8c", "fp16"), ("het4b", "fp32"), ("het8c", "q8"),
                                        ("aux_server", "fp16")])
def test_round_parity_lp_planned(fleet, wire):
    # the whole north-star chain on one GPU: spec -> solve_strategy ->
    # part_offsets -> GPU round with the LP's sample counts as weights
    from paper_2106_10207_b200.dist import plan_round
    from paper_2106_10207_b200.fleets import spec_json

    n = sum(RAGGED)
    plan = plan_round(spec_json(fleet), n, 4096 if wire == "q8" else 8)
    assert abs(sum(plan["fractions"]) - 1.0) < 1e-9
    _run_case(wire, plan["fractions"], plan["weights"], RAGGED, offsets=plan["offsets"])


@pytest.mark.parametrize("wire", ["fp32", "fp16", "q8"])
def test_round_parity_sharded_lamb_one_rank(wire):
    # shard_lamb on one rank: the owned range is the whole vector; exercises
    # the norm table, rank-ordered trust and the parameter push kernels
    _run_case(wire, [0.25, 0.25, 0.25, 0.25], [5.0, 0.0, 3.0, 8.0], RAGGED, steps=3, warm=True,
              shard=True)


def test_sharded_lamb_requires_param_buffer():
    n = sum(RAGGED)
    rnd = AveragingRound(n, RAGGED, wire="fp16", shard_lamb=True)
    rnd.assign([1.0], [1.0])
    g = torch.zeros(n, device="cuda")
    p, m, v = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    with pytest.raises(ValueError, match="param_ptr"):
        rnd.run([g], p, m, v, 1)
    rnd.run([g], rnd.param_buffer(), m, v, 1)
    torch.cuda.synchronize()
    rnd.close()
    r2 = AveragingRound(n, RAGGED, wire="fp16")
    with pytest.raises(RuntimeError):
        r2.param_buffer()
    r2.close()


@pytest.mark.parametrize("wire", ["fp16", "q8"])
def test_round_parity_multi_step_warm_state(wire):
    _run_case(wire, [0.25, 0.25, 0.25, 0.25], [5.0, 0.0, 3.0, 8.0], RAGGED, steps=3, warm=True)


@pytest.mark.parametrize("block", [512, 16384])
def test_round_parity_q8_block_sizes(block):
    _run_case("q8", [0.3, 0.7], [1.0, 2.0], RAGGED, block=block)


@pytest.mark.parametrize("wire,shard", [("fp16", False), ("q8", False), ("fp32", True)])
def test_lamb_tensor_larger_than_a_window(wire, shard):
    # a 9.5M-element tensor does not fit half the shared-memory stash (about
    # 4.3M elements on 148 SMs): it gets a window of its own, part of its
    # chunks stashed and the rest recomputed from p, m', v' in pass 2;
    # sharded on one rank: one window of 9.58M elements over the whole stash
    sizes = [3, 9_500_001, 70001, 5]
    _run_case(wire, [0.5, 0.5], [1.0, 3.0], sizes, steps=2, warm=True, shard=shard)


def test_lamb_plan_chunks():
    import json
    import os

    tables = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tensor_tables.json")))
    al = tables["albert-large"]
    rnd = AveragingRound(sum(al), al, wire="fp16")
    rnd.assign([1.0], [1.0])
    # chunks cut at every multiple of the tile and at every tensor edge
    n, tile = rnd.lamb_chunks()
    edges, start = set(), 0
    for sz in al:
        edges.update(range((start // tile + 1) * tile, start + sz, tile))
        edges.add(start)
        start += sz
    assert n == len(edges)
    rnd.close()
    rnd = AveragingRound(sum(al), al, wire="fp16", shard_lamb=True)
    rnd.assign([1.0], [1.0])
    assert rnd.lamb_chunks() == (n, tile)
    rnd.close()


def test_round_parity_albert_large_fp16_g8():
    import json
    import os

    tables = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tensor_tables.json")))
    _run_case("fp16", [1 / 8] * 8, [4.0] * 8, tables["albert-large"])


def test_phased_equals_graph():
    sizes = RAGGED
    n = sum(sizes)
    outs = []
    for phased in (False, True):
        g = torch.empty(n, device="cuda")
        fill_synthetic(g, 5, 0, SIGMA)
        g2 = torch.empty(n, device="cuda")
        fill_synthetic(g2, 5, 1, SIGMA)
        p = torch.full((n,), 0.01, device="cuda")
        m = torch.zeros(n, device="cuda")
        v = torch.zeros(n, device="cuda")
        rnd = AveragingRound(n, sizes, wire="fp16", peers_per_rank=2)
        rnd.assign([0.5, 0.5], [1.0, 3.0])
        for step in (1, 2):
            if phased:
                t = rnd.run_phased([g, g2], p, m, v, step)
                assert t["total_ms"] > 0
            else:
                rnd.run([g, g2], p, m, v, step)
        torch.cuda.synchronize()
        outs.append((p.cpu(), m.cpu(), v.cpu()))
        rnd.close()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("wire,shard", [("fp16", False), ("q8", False), ("fp32", True)])
def test_lamb_bits_do_not_depend_on_the_claim_order(wire, shard):
    # k_lamb hands chunks out at run time and runs pass 2 whenever a tensor
    # completes, so the chunk -> CTA map, the stash/recompute split and the
    # order of completions differ from launch to launch: the results must
    # not (norm partials per chunk, tensor sums in chunk order)
    import json
    import os

    sizes = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tensor_tables.json")))["albert-base"]
    n = sum(sizes)
    g = torch.empty(n, device="cuda")
    fill_synthetic(g, 9, 0, SIGMA)
    p0 = torch.empty(n, device="cuda")
    fill_synthetic(p0, 10, 0, 0.02, 0)
    rnd = AveragingRound(n, sizes, wire=wire, lr=HP["lr"], shard_lamb=shard)
    rnd.assign([1.0], [1.0])
    outs = []
    for _ in range(4):
        if shard:
            p = rnd.param_buffer()
            p.copy_(p0)
        else:
            p = p0.clone()
        m = torch.zeros(n, device="cuda")
        v = torch.zeros(n, device="cuda")
        for step in (1, 2, 3):
            rnd.run([g], p, m, v, step)
        torch.cuda.synchronize()
        outs.append((p.cpu().clone(), m.cpu(), v.cpu(), torch.tensor(rnd.read_trust())))
    rnd.close()
    for o in outs[1:]:
        for x, y in zip(outs[0], o):
            assert torch.equal(x, y)


def test_bad_arguments_raise():
    rnd = AveragingRound(1000, [1000], wire="fp16", peers_per_rank=2)
    with pytest.raises(ValueError):
        rnd.set_assignment([0, 3, 1000], [1.0, 1.0])  # inner offset not aligned
    with pytest.raises(ValueError):
        rnd.set_assignment([0, 504, 1000], [0.0, 0.0])  # sum of weights is zero
    p = torch.zeros(1000, device="cuda")
    with pytest.raises(RuntimeError):
        rnd.run([p, p], p, p, p, 1)  # before set_assignment
    rnd.close()


@pytest.mark.parametrize("wire", ["fp32", "fp16", "q8"])
def test_no_writes_outside_user_buffers(wire):
    """compute-sanitizer is closed on this pool: guard regions after p/m/v and
    around the gradients must survive rounds untouched (out-of-bounds writes
    into caller memory would show up here)."""
    sizes = [3, 1000, 70001, 2, 4096, 131075, 5]
    n, guard = sum(sizes), 4096
    sentinel = 12345.678

    def guarded(fill):
        t = torch.full((n + 2 * guard,), sentinel, device="cuda")
        t[guard:guard + n] = fill
        return t

    grads = []
    for g in range(4):
        t = torch.full((n + 2 * guard,), sentinel, device="cuda")
        fill_synthetic(t[guard:guard + n], 5, g, SIGMA)
        grads.append(t)
    p, m, v = guarded(0.02), guarded(0.0), guarded(0.0)
    rnd = AveragingRound(n, sizes, wire=wire, peers_per_rank=4)
    rnd.assign([0.1, 0.2, 0.3, 0.4], [1.0, 2.0, 3.0, 4.0])
    views = [g[guard:guard + n] for g in grads]
    for step in (1, 2, 3):
        rnd.run(views, p[guard:guard + n], m[guard:guard + n], v[guard:guard + n], step)
    rnd.run_phased(views, p[guard:guard + n], m[guard:guard + n], v[guard:guard + n], 4)
    torch.cuda.synchronize()
    for t in [p, m, v] + grads:
        assert torch.all(t[:guard] == sentinel) and torch.all(t[guard + n:] == sentinel)
    assert torch.isfinite(p[guard:guard + n]).all()
    rnd.close()


def _micro(n, seed, peer, k):
    return O.fill_synthetic(n, seed * 100 + k, peer, SIGMA)


@pytest.mark.parametrize("wire", ["fp16", "q8"])
def test_device_accumulation_weighted_by_sample_counts(wire):
    """Round step 1 on the device: peers accumulate micro-batches, the sample
    counts weight the average (per-peer counts 3, 1, 0, 5 micro-batches of 8,
    2, -, 4 samples), two rounds alternating the two buffers (DPU)."""
    sizes = RAGGED
    n = sum(sizes)
    G = 4
    plan = {0: [(k, 8.0) for k in range(3)], 1: [(0, 2.0)], 2: [], 3: [(k, 4.0) for k in range(5)]}
    rnd = AveragingRound(n, sizes, wire=wire, peers_per_rank=G, lr=HP["lr"], eps=HP["eps"],
                         weight_decay=HP["weight_decay"])
    rnd.assign([0.25] * 4, [1.0] * 4)  # weights unused by accumulated rounds
    p_h = O.fill_synthetic(n, 2, 0, 0.02, 0)
    m_h = np.zeros(n, np.float32)
    v_h = np.zeros(n, np.float32)
    p_d, m_d, v_d = _dev(p_h.copy()), _dev(m_h.copy()), _dev(v_h.copy())
    for step, buf in ((1, 0), (2, 1), (3, 0)):
        accs, counts = [], []
        for g in range(G):
            acc = None
            for k, smp in plan[g]:
                x = _micro(n, step, g, k)
                rnd.accumulate(g, _dev(x), smp, buf=buf)
                acc = x.copy() if acc is None else (acc + x).astype(np.float32)
            accs.append(acc)
            counts.append(sum(s for _, s in plan[g]))
            assert rnd.samples(g, buf) == counts[-1]
        rnd.run_accumulated(p_d, m_d, v_d, step, buf=buf)
        torch.cuda.synchronize()
        assert rnd.samples(0, buf) == 0.0  # counts reset after the round
        packed = [None if a is None else O.pack(wire, a) for a in accs]
        wires = [np.zeros(1, np.float32) if q is None else q[0] for q in packed]
        scales = [None if q is None else q[1] for q in packed]
        avg, avg_s = O.reduce(wire, wires, scales, counts, 0, n, n)
        got, gs = rnd.read_wire(nat.SP_BUF_AVG)
        np.testing.assert_array_equal(got, avg)
        if wire == "q8":
            np.testing.assert_array_equal(gs, avg_s)
        trust = rnd.read_trust()
        O.lamb(wire, avg, avg_s, p_h, m_h, v_h, sizes, HP, step, trust_in=trust)
        np.testing.assert_array_equal(p_d.cpu().numpy(), p_h)
        np.testing.assert_array_equal(m_d.cpu().numpy(), m_h)
    # writing gradients in place through the accumulator view
    acc0 = rnd.accumulator(0, buf=1)
    acc0.copy_(_dev(_micro(n, 9, 0, 0)))
    rnd.add_samples(0, 6.0, buf=1)
    assert rnd.samples(0, buf=1) == 6.0
    rnd.close()


def test_measured_round_times_feed_compare_strategies():
    # each algorithm's partition run on the executor and timed
    import json

    from golden.fleets import spec
    from paper_2106_10207_b200.measure import compare_strategies_measured

    s = spec("het4b")
    s["param_count"] = 1_000_000
    rows = {r["algorithm"]: r for r in compare_strategies_measured(json.dumps(s), steps=5)}
    assert set(rows) == {"allreduce", "parameter_server", "adaptive"}
    for r in rows.values():
        assert 0 < r["measured_round_s"] < 0.1
        assert r["round_s"] == r["measured_round_s"]
        assert r["steps_per_hour"] > 0


@pytest.mark.parametrize("wire", ["fp16", "q8"])
def test_dpu_overlap_accumulate_during_round(wire):
    """SURVEY §8f N4 (the reference models it as
    max(compute, comm), netsim.cpp:291-293): step s's round runs on one
    stream while step s+1's micro-batches accumulate into the other buffer on
    a second stream. The result is bit-identical to the serial schedule."""
    sizes = RAGGED
    n = sum(sizes)
    G, steps = 2, 4
    micro = {(s, g, k): _dev(_micro(n, s, g, k)) for s in range(1, steps + 2) for g in range(G)
             for k in range(g + 1)}
    torch.cuda.synchronize()

    def fresh():
        rnd = AveragingRound(n, sizes, wire=wire, peers_per_rank=G, lr=HP["lr"], eps=HP["eps"],
                             weight_decay=HP["weight_decay"])
        rnd.assign([0.5, 0.5], [1.0, 1.0])
        p = _dev(O.fill_synthetic(n, 2, 0, 0.02, 0))
        return rnd, p, torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")

    def acc(rnd, s, stream):
        for g in range(G):
            for k in range(g + 1):
                rnd.accumulate(g, micro[(s, g, k)], 4.0 + g, buf=s % 2, stream=stream)

    # serial: accumulate, then round, one stream
    rnd, p1, m1, v1 = fresh()
    for s in range(1, steps + 1):
        acc(rnd, s, None)
        rnd.run_accumulated(p1, m1, v1, s, buf=s % 2)
    torch.cuda.synchronize()
    rnd.close()
    # overlapped: round s on stream A || accumulation of s+1 on stream B
    rnd, p2, m2, v2 = fresh()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    acc(rnd, 1, sb)
    done = {}
    for s in range(1, steps + 1):
        sa.wait_stream(sb)  # step s's accumulators are complete
        rnd.run_accumulated(p2, m2, v2, s, buf=s % 2, stream=sa)
        done[s] = torch.cuda.Event()
        done[s].record(sa)
        if s < steps:
            if s - 1 in done:  # round s-1 has finished reading the buffer s+1 reuses
                sb.wait_event(done[s - 1])
            acc(rnd, s + 1, sb)  # the other buffer, concurrently with round s
    torch.cuda.synchronize()
    rnd.close()
    for a, b in ((p1, p2), (m1, m2), (v1, v2)):
        assert torch.equal(a, b)


@pytest.mark.parametrize("wire,shard", [("fp16", False), ("q8", False), ("fp32", True)])
def test_run_host_matches_device_round(wire, shard):
    # sp_round_run_host: pinned host gradients, double-buffered staging on a
    # copy stream (two cached graphs); must equal sp_round_run bit for bit
    sizes = RAGGED
    n = sum(sizes)
    G = 2
    fr, w = [0.5, 0.5], [3.0, 5.0]
    outs = []
    for use_host in (False, True):
        rnd = AveragingRound(n, sizes, wire=wire, peers_per_rank=G, lr=HP["lr"], eps=HP["eps"],
                             weight_decay=HP["weight_decay"], shard_lamb=shard)
        rnd.assign(fr, w)
        p = rnd.param_buffer() if shard else torch.empty(n, device="cuda")
        fill_synthetic(p, 5, 0, 0.02, 0)
        m = torch.zeros(n, device="cuda")
        v = torch.zeros(n, device="cuda")
        for step in range(1, 5):  # different gradients every step
            grads = []
            for g in range(G):
                t = torch.empty(n, device="cuda")
                fill_synthetic(t, 40 + step, g, SIGMA)
                grads.append(t)
            if use_host:
                hg = [t.cpu().pin_memory() for t in grads]
                torch.cuda.synchronize()
                rnd.run_host(hg, p, m, v, step)
                del grads
            else:
                rnd.run(grads, p, m, v, step)
            torch.cuda.synchronize()
        outs.append([x.cpu().numpy().copy() for x in (p, m, v)])
        rnd.close()
    for a, b, name in zip(outs[0], outs[1], "pmv"):
        np.testing.assert_array_equal(a, b, err_msg=name)


# ----------------------------------------------------------------------------
# BASELINE.json configs 1-4 at full size (virtual peers on one GPU), the
# averaged vector against the REFERENCE's own run_plan (oracle/_ref: the
# fp64 weighted mean of groups.cpp:117-161 over the dequantized wire inputs).
# Tolerance, elementwise, with a_g = (w_g / W) |x_g|:
#   fp32 accumulation of G fmaf terms with fp32 weights: (G + 2) 2^-24 sum_g a_g
#   plus the output's wire rounding: fp32 none, fp16 2^-11 |mean| + 2^-25,
#   q8 half a code step of the output block (scale / 2).
FULL_SIZE = {
    "het4b-albert-base-fp32": ("albert-base", "fp32", "het4b"),
    "g8-albert-large-fp16": ("albert-large", "fp16", None),
    "g8-resnet50-q8": ("resnet50", "q8", None),
    "het8c-albert-large-fp16": ("albert-large", "fp16", "het8c"),
}


@pytest.mark.parametrize("name", sorted(FULL_SIZE))
def test_full_size_average_vs_reference_run_plan(name):
    import json
    import os

    from oracle import ref as R
    from paper_2106_10207_b200.dist import plan_round
    from paper_2106_10207_b200.fleets import homogeneous, spec_json

    table, wire, fleet = FULL_SIZE[name]
    tables = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tensor_tables.json")))
    sizes = tables[table]
    n = sum(sizes)
    block = 4096
    sj = spec_json(fleet) if fleet else json.dumps(homogeneous(8, 1.0, 1000.0, 4096.0, n))
    plan = plan_round(sj, n, block if wire == "q8" else 8)
    G = len(plan["fractions"])
    weights = plan["weights"]
    grads = []
    for g in range(G):
        t = torch.empty(n, device="cuda")
        fill_synthetic(t, 7, g, SIGMA)
        grads.append(t)
    p = torch.zeros(n, device="cuda")
    m, v = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    rnd = AveragingRound(n, sizes, wire=wire, q8_block=block, peers_per_rank=G)
    rnd.set_assignment(plan["offsets"], weights)
    rnd.run(grads, p, m, v, 1)
    torch.cuda.synchronize()
    got_w, got_s = rnd.read_wire(nat.SP_BUF_AVG)
    rnd.close()
    del grads
    got = O.dequant(wire, got_w, got_s, block)
    # the reference's weighted mean of what each peer put on the wire
    wires = []
    for g in range(G):
        x = O.fill_synthetic(n, 7, g, SIGMA)
        q = O.pack(wire, x, block)
        wires.append(None if weights[g] == 0 else O.dequant(wire, q[0], q[1], block))
    want = R.weighted_mean(wires, weights)
    W = sum(weights)
    acc_mag = np.zeros(n, np.float64)
    for g in range(G):
        if wires[g] is not None:
            acc_mag += (weights[g] / W) * np.abs(wires[g].astype(np.float64))
    tol = (G + 2) * 2.0 ** -24 * acc_mag
    if wire == "fp16":
        tol += 2.0 ** -11 * np.abs(want) + 2.0 ** -25
    elif wire == "q8":
        tol += np.repeat(got_s.astype(np.float64), block)[:n] / 2 * (1 + 1e-6)
    err = np.abs(got.astype(np.float64) - want)
    bad = err > tol
    assert not bad.any(), (f"{int(bad.sum())} elements outside tolerance; worst at "
                           f"{int(np.argmax(err - tol))}: got {got[np.argmax(err - tol)]}, "
                           f"want {want[np.argmax(err - tol)]}")
