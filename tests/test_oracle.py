"""CPU oracle checks (no GPU): the oracle is pinned to the reference's known
answers where the reference has any, and to independent numpy restatements
where the arithmetic is framework-defined."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2106_10207_b200.round import part_offsets


# --------------------------------------------------------------- run_plan
def test_weighted_average_spec_known_answers():
    # SPEC.md:246 "n=4, m=2, no failures, inputs [0,0,0,4] -> all peers 1.0"
    vals = [np.array([x], np.float64) for x in (0, 0, 0, 4)]
    assert O.weighted_average_f64(vals, None)[0] == 1.0
    # SPEC.md:219 "n=9, m=3 -> averaging inputs [1..9] yields 5.0"
    vals = [np.array([x], np.float64) for x in range(1, 10)]
    assert O.weighted_average_f64(vals, None)[0] == 5.0


def test_weighted_average_matches_run_plan_semantics():
    # groups.cpp:119-120,143-144,158: sum_i (w_i v_i) in peer order, / sum w
    rng = np.random.default_rng(3)
    vals = [rng.standard_normal(257) for _ in range(5)]
    w = [3.0, 0.0, 1.0, 7.0, 2.5]
    out = O.weighted_average_f64(vals, w)
    s = np.zeros(257)
    for v, wi in zip(vals, w):
        s = s + v * wi
    np.testing.assert_array_equal(out, s / sum(w))


# -------------------------------------------------------------- synthetic
def _splitmix64(x):
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return x ^ (x >> 31)


def test_synthetic_generator_restated_in_python():
    n, seed, peer, scale = 2000, 1, 3, np.float32(1e-3 * np.sqrt(3.0))
    got = O.fill_synthetic(n, seed, peer, float(scale), 997, 100.0)
    key = seed ^ (peer << 40)
    for i in range(0, n, 37):
        u = _splitmix64(key ^ i) >> 40
        x = np.float32(np.float32(u) - np.float32(8388608.0)) * np.float32(1.0 / 8388608.0)
        x = np.float32(x * scale)
        if i % 997 == 0:
            x = np.float32(x * np.float32(100.0))
        assert got[i] == x, i
    assert np.abs(got).max() <= 100 * float(scale) * 1.0001


# ------------------------------------------------------------------- fp16
def test_f2h_matches_numpy_rne():
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2**32, 200000, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[np.isfinite(x)]
    edge = np.array([0.0, -0.0, 65504.0, 65519.99, 65520.0, 1e30, -1e30, 2**-24, 2**-25,
                     2**-25 * 1.0000001, 3 * 2**-26, 6.1e-5, 5.96e-8, 1.0 + 2**-11,
                     1.0 + 3 * 2**-11, np.inf, -np.inf], np.float32)
    for arr in (x, edge, (rng.standard_normal(100000) * 1e-3).astype(np.float32),
                (rng.standard_normal(100000) * 1e-6).astype(np.float32)):
        np.testing.assert_array_equal(O.pack_fp16(arr), arr.astype(np.float16).view(np.uint16))


# --------------------------------------------------------------------- q8
def _q8_numpy(x, block):
    codes = np.zeros(x.size, np.int8)
    scales = np.zeros((x.size + block - 1) // block, np.float32)
    for b in range(scales.size):
        blk = x[b * block:(b + 1) * block]
        amax = np.float32(np.abs(blk).max())
        inv = np.float32(np.float32(127.0) / amax) if amax > 0 else np.float32(0)
        q = np.rint((blk * inv).astype(np.float32))
        codes[b * block:(b + 1) * block] = np.clip(q, -127, 127).astype(np.int8)
        scales[b] = np.float32(amax / np.float32(127.0))
    return codes, scales


@pytest.mark.parametrize("block", [512, 4096])
def test_q8_matches_numpy_restatement(block):
    x = O.fill_synthetic(3 * block + 123, 7, 0, 1e-3)
    x[block:2 * block] = 0.0  # an all-zero block
    c, s = O.pack_q8(x, block)
    c2, s2 = _q8_numpy(x, block)
    np.testing.assert_array_equal(c, c2)
    np.testing.assert_array_equal(s, s2)
    assert s[1] == 0 and not c[block:2 * block].any()
    deq = O.dequant("q8", c, s, block)
    err = np.abs(deq - x)
    bound = np.repeat(s, block)[: x.size] * 0.5000001 + 1e-12
    assert (err <= bound).all()


# ----------------------------------------------------------------- reduce
@pytest.mark.parametrize("wire", ["fp32", "fp16", "q8"])
def test_reduce_close_to_fp64_weighted_mean(wire):
    n, G, block = 3 * 4096 + 77, 4, 4096
    grads = [O.fill_synthetic(n, 1, g, 1e-3) for g in range(G)]
    w = [5.0, 1.0, 0.0, 2.0]
    packed = [O.pack(wire, g, block) for g in grads]
    out, osc = O.reduce(wire, [p[0] for p in packed], [p[1] for p in packed], w, 0, n, n, block)
    got = O.dequant(wire, out, osc, block)
    deq_in = [O.dequant(wire, p[0], p[1], block).astype(np.float64) for p in packed]
    ref = O.weighted_average_f64(deq_in, w)
    tol = {"fp32": 1e-6, "fp16": 2.0**-11, "q8": 1 / 127.0}[wire]
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= tol * scale


@pytest.mark.parametrize("wire", ["fp32", "fp16", "q8"])
def test_reduce_single_contributor_is_identity(wire):
    # one nonzero weight: the average is that peer's wire values, unchanged
    # (q8 by definition: codes and scales forwarded, no requantization)
    n, block = 5 * 4096 + 300, 4096
    packed = [O.pack(wire, O.fill_synthetic(n, 3, g, 1e-3, 997, 100.0), block) for g in range(3)]
    out, osc = O.reduce(wire, [p[0] for p in packed], [p[1] for p in packed], [0.0, 7.0, 0.0],
                        0, n, n, block)
    np.testing.assert_array_equal(out, packed[1][0][:n])
    if wire == "q8":
        np.testing.assert_array_equal(osc, packed[1][1])


def test_q8_requantize_keeps_codes():
    # why forwarding is the right definition: requantizing a peer's dequantized
    # block reproduces every code; only the scale may move by an ulp
    n, block = 8 * 4096, 4096
    c, s = O.pack_q8(O.fill_synthetic(n, 4, 0, 1e-3, 997, 100.0), block)
    deq = O.dequant("q8", c, s, block)
    c2, s2 = O.pack_q8(deq, block)
    np.testing.assert_array_equal(c, c2)
    assert np.all(np.abs(s2.view(np.int32) - s.view(np.int32)) <= 1)


# ------------------------------------------------------------------- LAMB
def _lamb_numpy(g, p, m, v, sizes, hp, step):
    p, m, v = p.astype(np.float64), m.astype(np.float64), v.astype(np.float64)
    g = g.astype(np.float64)
    b1, b2 = hp["beta1"], hp["beta2"]
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh, vh = m / (1 - b1**step), v / (1 - b2**step)
    u = mh / (np.sqrt(vh) + hp["eps"]) + hp["weight_decay"] * p
    out, off = p.copy(), 0
    for s in sizes:
        sl = slice(off, off + s)
        r1, r2 = np.linalg.norm(p[sl]), np.linalg.norm(u[sl])
        tr = r1 / r2 if r1 > 0 and r2 > 0 else 1.0
        out[sl] = p[sl] - hp["lr"] * tr * u[sl]
        off += s
    return out, m, v


HP = dict(lr=1.76e-3, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.01, bias_correction=1)


@pytest.mark.parametrize("step", [1, 7])
def test_lamb_close_to_float64_numpy(step):
    sizes = [3, 1000, 70001, 2, 4096]
    n = sum(sizes)
    g = O.fill_synthetic(n, 2, 0, 1e-3)
    p = O.fill_synthetic(n, 3, 0, 0.02)
    m = O.fill_synthetic(n, 4, 0, 1e-4)
    v = np.abs(O.fill_synthetic(n, 5, 0, 1e-6))
    pr, mr, vr = _lamb_numpy(g, p, m, v, sizes, HP, step)
    trust = O.lamb("fp32", g, None, p, m, v, sizes, HP, step)
    assert (trust > 0).all()
    # fp32 arithmetic vs fp64: errors relative to each array's scale
    for got, ref in ((m, mr), (v, vr), (p, pr)):
        assert np.abs(got - ref).max() <= 2e-6 * np.abs(ref).max()


def test_lamb_trust_is_one_for_zero_params():
    sizes = [100]
    g = O.fill_synthetic(100, 2, 0, 1e-3)
    p = np.zeros(100, np.float32)
    m = np.zeros(100, np.float32)
    v = np.zeros(100, np.float32)
    hp = dict(HP, weight_decay=0.0)
    trust = O.lamb("fp32", g, None, p, m, v, sizes, hp, 1)
    assert trust[0] == 1.0


# ------------------------------------------------------------- partitions
HET8C = [1 / 20] * 6 + [0.0, 7 / 10]
HET4B = [1 / 22] * 3 + [19 / 22]


@pytest.mark.parametrize("fr", [HET8C, HET4B, [1 / 8] * 8, [1.0], [0.0, 1.0, 0.0]])
@pytest.mark.parametrize("align", [8, 4096])
def test_part_offsets_oracle_equals_host(fr, align):
    for n in (17847474, 11813810, 25557032, 1000, 7):
        a = O.part_offsets(n, fr, align)
        b = part_offsets(n, fr, align)
        assert a == b
        assert a[0] == 0 and a[-1] == n
        assert all(x <= y for x, y in zip(a, a[1:]))
        assert all(x % align == 0 for x in a[1:-1] if x < n)


def test_part_offsets_het8c_shape():
    offs = part_offsets(17847474, HET8C, 8)
    lens = [b - a for a, b in zip(offs, offs[1:])]
    assert lens[6] == 0  # the client owns nothing
    assert abs(lens[7] / 17847474 - 0.7) < 1e-5


def test_part_offsets_round_half_away_exactly():
    # x = n * cum / align just below 0.5: llround gives 0, floor(x + 0.5)
    # would give 1; the Python mirror, the C++ partitioner and
    # the C oracle agree
    from paper_2106_10207_b200 import _swarmplan as sp

    f = 0.49999999999999994
    for n, fr, align in [(1, [f, 1 - f], 1), (2, [f / 2, 1 - f / 2], 1), (8, [f / 8 * 8, 1.0], 8)]:
        want = sp.part_offsets(n, fr, align)
        assert part_offsets(n, fr, align) == want == O.part_offsets(n, fr, align), (n, fr)
    assert part_offsets(1, [f, 1 - f], 1) == [0, 0, 1]
