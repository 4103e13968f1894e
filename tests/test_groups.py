"""Group plans and the CPU averaging executor (swarmplan::groups via the
binding). The reference's test_groups.cpp is an empty stub, so these encode
SPEC.md's examples and invariants for the module and the
run_plan <-> oracle identity for the butterfly case (m = n). Parity with the
reference's own compiled run_plan is in tests/test_ref_pin.py; the GPU
executor is checked against it here."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2106_10207_b200 import _swarmplan as sp


def _rounds(n, m):
    r, reach = 0, 1
    while reach < n:
        reach *= m
        r += 1
    return r


@pytest.mark.parametrize("n", list(range(1, 40)) + [64])
def test_plan_shape_and_exactness(n):
    rng = np.random.default_rng(n)
    vals = rng.standard_normal((n, 7))
    for m in range(2, max(n, 2) + 1):
        plan = sp.build_plan(n, m)
        assert len(plan) == _rounds(n, m)
        for groups in plan:
            members = sorted(p for g in groups for p in g)
            assert members == list(range(n))
        # SPEC.md:240-241 exactness holds for the exact merge rule; the
        # reference's rule (the default) double-counts on some ragged plans
        res = sp.run_plan(n, m, vals, exact=True)
        np.testing.assert_allclose(res["values"], np.broadcast_to(vals.mean(0), vals.shape),
                                   rtol=1e-9, atol=1e-12)
        assert all(res["complete"]) and res["groups_failed"] == 0


def test_spec_examples():
    # SPEC.md:219-221
    plan = sp.build_plan(9, 3)
    assert len(plan) == 2
    res = sp.run_plan(9, 3, np.arange(1.0, 10.0).reshape(9, 1))
    assert (res["values"] == 5.0).all()
    assert sp.build_plan(4, 4) == [[[0, 1, 2, 3]]]
    assert len(sp.build_plan(6, 2)) == 3
    # SPEC.md:246
    res = sp.run_plan(4, 2, np.array([[0.0], [0.0], [0.0], [4.0]]))
    assert (res["values"] == 1.0).all()
    assert len(sp.build_plan(16, 4)) == 2  # test_smoke.py:58-62


def test_failed_group_is_isolated():
    # a failure only affects the immediate group
    vals = np.array([[1.0], [2.0], [3.0], [4.0]])
    plan = sp.build_plan(4, 2)
    failing = plan[0].index([2, 3]) if [2, 3] in plan[0] else 1
    res = sp.run_plan(4, 2, vals, [], [(0, failing)])
    assert res["groups_failed"] == 1
    assert not all(res["complete"])
    ok_group = plan[0][1 - failing]
    # members of the healthy group progressed in round 0 (coverage >= 2)
    assert all(res["coverage"][p] >= 2 for p in ok_group)


def test_weighted_butterfly_equals_oracle_bit_for_bit():
    # m = n: one group, classes merged in peer order (groups.cpp:133-144)
    rng = np.random.default_rng(5)
    n, dim = 8, 1000
    vals = rng.standard_normal((n, dim))
    w = [float(x) for x in rng.integers(0, 50, n)]
    w[3] = 0.0
    res = sp.run_plan(n, n, vals, w)
    ref = O.weighted_average_f64(list(vals), w)
    for i in range(n):
        np.testing.assert_array_equal(res["values"][i], ref)


def test_bad_arguments():
    with pytest.raises(ValueError):
        sp.build_plan(0, 2)
    with pytest.raises(ValueError):
        sp.build_plan(4, 5)
    with pytest.raises(ValueError):
        sp.run_plan(4, 2, np.zeros((3, 2)))
    with pytest.raises(ValueError):
        sp.run_plan(4, 2, np.zeros((4, 2)), [1.0, 2.0])


def test_expected_iterations_and_group_size():
    assert sp.expected_iterations(16, 16, 0.0) == pytest.approx(1.0)
    for n, m in [(9, 3), (16, 2), (10, 4)]:
        assert sp.expected_iterations(n, m, 0.0) == pytest.approx(_rounds(n, m))
    for n in range(4, 65):
        assert sp.optimal_group_size(n, 0.0) == n
    assert sp.optimal_group_size(16, 0.5) == 2
    prev = 10**9
    for p in np.linspace(0.0, 0.4, 9):  # larger p: the 5e7-term series limit (domain_error)
        m = sp.optimal_group_size(24, float(p))
        assert m <= prev
        prev = m
    with pytest.raises(ValueError):
        sp.expected_iterations(4, 2, 1.0)


def test_expected_iterations_monte_carlo():
    rng = np.random.default_rng(0)
    n, m, p, trials = 16, 2, 0.3, 200000
    groups = math.ceil(n / m)
    q = (1 - p) ** m
    draws = rng.geometric(q, size=(trials, groups)).max(1)
    est = _rounds(n, m) * draws.mean()
    se = _rounds(n, m) * draws.std() / math.sqrt(trials)
    assert abs(sp.expected_iterations(n, m, p) - est) < 3 * se + 1e-9


def test_run_plan_device_rejects_bad_rows():
    # argument checks happen before any device work (CPU-safe)
    with pytest.raises(ValueError):
        sp.run_plan_device(4, 2, [0, 0, 0], 8, [0, 0, 0, 0])


GPU_CASES = [(4, 2, []), (5, 2, []), (9, 3, []), (16, 4, []), (13, 5, []), (8, 8, []),
             (6, 2, [(0, 1)]), (9, 3, [(1, 0)]), (16, 2, [(0, 3), (2, 1)]), (10, 4, [(0, 0), (1, 2)])]


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,failures", GPU_CASES)
@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("exact", [False, True])
def test_run_plan_gpu_bit_exact(n, m, failures, weighted, exact):
    # default rule: against the reference's own compiled run_plan
    # (oracle/_ref); exact rule: against the CPU executor's exact mode
    import torch

    from oracle import ref as R
    from paper_2106_10207_b200.groups import run_plan_gpu

    rng = np.random.default_rng(n * 100 + m)
    dim = 4097
    vals = rng.standard_normal((n, dim))
    w = [float(x) for x in rng.integers(0, 9, n)] if weighted else []
    if weighted:
        w[0] = max(w[0], 1.0)
    ref = sp.run_plan(n, m, vals, w, failures, exact=True) if exact else R.run_plan(n, m, vals, w, failures)
    got = run_plan_gpu(n, m, torch.from_numpy(vals).cuda(), w, failures, exact=exact)
    torch.cuda.synchronize()
    g = got["values"].cpu().numpy()
    # 0/0 (an all-zero-weight class) gives NaN on both sides
    np.testing.assert_array_equal(g, ref["values"])
    assert got["complete"] == ref["complete"]
    assert got["coverage"] == ref["coverage"]
    assert got["groups_failed"] == ref["groups_failed"]
