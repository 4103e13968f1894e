"""LP core (swarmplan::lp via the binding) — ports of
/root/reference/proj/tests/cpp/test_lp.cpp (unit cases :130-239, row scaling
:252-269, the 200-case vertex-enumeration oracle :271-290) plus scipy HiGHS
on larger random programs. Warm-start cases need the C++ class API and live
in tests/cpp/test_lp_warm.cpp (run by test_cpp_unit.py)."""
import itertools
import math

import numpy as np
import pytest
from scipy.optimize import linprog

from paper_2106_10207_b200 import _swarmplan as sp

INF = math.inf


def solve(nv, obj, lo, up, rows):
    return sp.lp_solve(nv, list(obj), list(lo), list(up), rows)


def test_single_bounded_variable():
    r = solve(1, [1.0], [0.0], [10.0], [([(0, 1.0)], "<=", 3.0)])
    assert r["status"] == "optimal" and r["objective"] == pytest.approx(3.0)
    assert r["x"][0] == pytest.approx(3.0)


def test_ties_across_optimal_face():
    r = solve(2, [1, 1], [0, 0], [1, 1], [([(0, 1.0), (1, 1.0)], "<=", 1.0)])
    assert r["objective"] == pytest.approx(1.0) and r["violation"] <= 1e-7


def test_equality_rows():
    r = solve(2, [1, -1], [0, 0], [2, 2], [([(0, 1.0), (1, 1.0)], "=", 0.5)])
    assert r["objective"] == pytest.approx(0.5)
    assert r["x"][0] + r["x"][1] == pytest.approx(0.5)


def test_infeasible():
    assert solve(1, [1], [0], [INF], [([(0, 1.0)], "<=", -1.0)])["status"] == "infeasible"
    assert solve(2, [0, 0], [0, 0], [1, 1], [([(0, 1.0), (1, 1.0)], "=", 5.0)])["status"] == "infeasible"


def test_unbounded():
    assert solve(2, [1, 0], [0, 0], [INF, INF], [([(1, 1.0)], "<=", 1.0)])["status"] == "unbounded"


def test_malformed_programs_rejected():
    with pytest.raises(ValueError):
        solve(2, [0, 0, 0], [0, 0], [INF, INF], [])  # objective size
    with pytest.raises(ValueError):
        solve(1, [0], [2.0], [1.0], [])  # lo > hi
    with pytest.raises(ValueError):
        solve(1, [0], [0], [INF], [([(3, 1.0)], "<=", 1.0)])  # unknown var
    with pytest.raises(ValueError):
        solve(1, [0], [0], [INF], [([(0, 1.0)], "<=", math.nan)])
    with pytest.raises(ValueError):
        solve(1, [0], [0], [INF], [([(0, INF)], "<=", 1.0)])


def _random_box_lp(seed):
    rng = np.random.default_rng(seed)
    nv = 2 + int(rng.integers(0, 3))
    nr = 1 + int(rng.integers(0, 5))
    up = [float(0.5 + 2.5 * rng.uniform()) for _ in range(nv)]
    obj = [float(2 * rng.uniform() - 1) for _ in range(nv)]
    rows = []
    for r in range(nr):
        co = [(j, float(4 * rng.uniform() - 2)) for j in range(nv) if rng.uniform() < 0.8] or [(0, 1.0)]
        rel = "=" if (r == 0 and seed % 5 == 0) else "<="
        rows.append((co, rel, float(4 * rng.uniform())))
    return nv, obj, up, rows


def _vertex_oracle(nv, obj, up, rows):
    """Brute force over active sets (test_lp.cpp:25-103)."""
    forced, optional = [], []
    for co, rel, rhs in rows:
        a = np.zeros(nv)
        for j, c in co:
            a[j] += c
        (forced if rel == "=" else optional).append((a, rhs))
    for j in range(nv):
        e = np.zeros(nv)
        e[j] = 1.0
        optional += [(e, 0.0), (e, up[j])]
    need = nv - len(forced)
    best = None
    for pick in itertools.combinations(range(len(optional)), need):
        M = np.array([f[0] for f in forced] + [optional[i][0] for i in pick])
        b = np.array([f[1] for f in forced] + [optional[i][1] for i in pick])
        if abs(np.linalg.det(M)) < 1e-12:
            continue
        x = np.linalg.solve(M, b)
        ok = all(x[j] >= -1e-9 and x[j] <= up[j] + 1e-9 for j in range(nv))
        for co, rel, rhs in rows:
            lhs = sum(c * x[j] for j, c in co)
            scale = max(abs(c) for _, c in co) or 1.0
            gap = (lhs - rhs) / scale
            ok = ok and (abs(gap) <= 1e-7 if rel == "=" else gap <= 1e-7)
        if ok:
            v = float(np.dot(obj, x))
            best = v if best is None else max(best, v)
    return best


def test_vertex_enumeration_oracle_200_programs():
    infeasible = 0
    for seed in range(1, 201):
        nv, obj, up, rows = _random_box_lp(seed)
        best = _vertex_oracle(nv, obj, up, rows)
        r = solve(nv, obj, [0.0] * nv, up, rows)
        if best is None:
            infeasible += 1
            assert r["status"] == "infeasible", seed
            continue
        assert r["status"] == "optimal", seed
        assert r["objective"] == pytest.approx(best, rel=1e-7, abs=1e-7 * max(1.0, best)), seed
        assert r["violation"] <= 1e-6, seed
    assert infeasible > 0


def test_repeat_solves_bit_identical():
    nv, obj, up, rows = _random_box_lp(424242)
    assert solve(nv, obj, [0.0] * nv, up, rows) == solve(nv, obj, [0.0] * nv, up, rows)


def test_row_scaling_does_not_move_optimum():
    rows = [([(0, 1.0), (1, 1.0)], "<=", 2.0), ([(1, 1.0), (2, 2.0)], "<=", 3.0)]
    base = solve(3, [3, 1, 2], [0] * 3, [5] * 3, rows)
    scaled = solve(3, [3, 1, 2], [0] * 3, [5] * 3,
                   [([(j, c * 1e3) for j, c in co], rel, rhs * 1e3) for co, rel, rhs in rows])
    assert scaled["objective"] == pytest.approx(base["objective"], rel=1e-9)
    np.testing.assert_allclose(scaled["x"], base["x"], rtol=1e-9)


@pytest.mark.parametrize("seed", range(40))
def test_matches_highs_on_larger_programs(seed):
    rng = np.random.default_rng(1000 + seed)
    nv, nr = int(rng.integers(10, 60)), int(rng.integers(5, 50))
    A = rng.uniform(-1, 2, (nr, nv)) * (rng.uniform(size=(nr, nv)) < 0.3)
    b = rng.uniform(0.5, 5, nr)
    up = rng.uniform(0.5, 4, nv)
    obj = rng.uniform(-1, 1, nv)
    rows = [([(j, float(A[i, j])) for j in range(nv) if A[i, j] != 0] or [(0, 1.0)], "<=", float(b[i]))
            for i in range(nr)]
    A2 = np.array([[dict(co).get(j, 0.0) for j in range(nv)] for co, _, _ in rows])
    ref = linprog(-obj, A_ub=A2, b_ub=b, bounds=list(zip([0] * nv, up)), method="highs")
    r = solve(nv, obj, [0.0] * nv, up, rows)
    assert r["status"] == "optimal"
    assert r["objective"] == pytest.approx(-ref.fun, rel=1e-8, abs=1e-8)
    assert r["violation"] <= 1e-7
