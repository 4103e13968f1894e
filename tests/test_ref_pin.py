"""Parity of the host code with the REFERENCE ITSELF: oracle/_ref is the
reference's own groups.cpp and model.cpp compiled unmodified
(oracle/build_ref.py). These pin

  * groups::build_plan for every n <= 64 and every group size m,
  * groups::run_plan bit for bit (values, complete, coverage, groups_failed)
    for every n <= 40 and m, with weights and failed groups, ragged plans
    included (the reference's merge rule, groups.cpp:126-151),
  * spec parsing / validation / JSON output (model.cpp:38-205) on the
    fixtures and on a corpus of mutated specs, messages included.

CPU only; skipped when neither /root/reference nor a prebuilt
oracle/_ref/libswarmplan_ref.so is present.
"""
import copy
import json
import os

import numpy as np
import pytest

from golden.fleets import FLEETS, homogeneous, spec_json
from paper_2106_10207_b200 import _swarmplan as sp

ref = pytest.importorskip("oracle.ref")
if not ref.available():
    pytest.skip("oracle/_ref not built and /root/reference absent", allow_module_level=True)

SCENARIOS = "/root/reference/proj/scenarios"


def test_build_plan_matches_reference_all_n_m():
    for n in range(1, 65):
        for m in range(2, max(n, 2) + 1):
            assert sp.build_plan(n, m) == ref.build_plan(n, m), (n, m)


@pytest.mark.parametrize("n,m", [(0, 2), (4, 1), (4, 5), (1, 3), (-1, 2)])
def test_build_plan_errors_match_reference(n, m):
    with pytest.raises(ValueError) as a:
        sp.build_plan(n, m)
    with pytest.raises(ValueError) as b:
        ref.build_plan(n, m)
    assert str(a.value) == str(b.value)


def _same_result(a, b):
    np.testing.assert_array_equal(a["values"], b["values"])  # NaN == NaN here
    assert list(a["complete"]) == list(b["complete"])
    assert list(a["coverage"]) == list(b["coverage"])
    assert a["groups_failed"] == b["groups_failed"]


def test_run_plan_matches_reference_bit_for_bit():
    rng = np.random.default_rng(2106)
    for n in range(1, 41):
        for m in range(2, max(n, 2) + 1):
            vals = rng.standard_normal((n, 5)) * 10.0 ** rng.integers(-3, 4, (n, 1))
            plan = sp.build_plan(n, m)
            cases = [([], [])]
            w = [float(x) for x in rng.integers(0, 9, n)]
            w[rng.integers(n)] = 1.0 + rng.random()
            cases.append((w, []))
            if plan:
                fails = {(int(r), int(rng.integers(len(plan[r])))) for r in rng.integers(0, len(plan), 2)}
                cases.append((w, sorted(fails)))
            for weights, failures in cases:
                got = sp.run_plan(n, m, vals, weights, failures)
                want = ref.run_plan(n, m, vals, weights, failures)
                _same_result(got, want)


def test_ragged_double_count_is_the_reference_behaviour():
    # n = 5, m = 2, inputs 1..5: the reference's rule counts one partial sum
    # twice on some peers (2.7778 instead of 3); run_plan keeps that
    # behaviour by default and exact=True gives SPEC.md:240-241's mean
    vals = np.arange(1.0, 6.0).reshape(5, 1)
    want = ref.run_plan(5, 2, vals)
    got = sp.run_plan(5, 2, vals)
    _same_result(got, want)
    assert not np.allclose(want["values"], 3.0)
    exact = sp.run_plan(5, 2, vals, exact=True)
    np.testing.assert_allclose(exact["values"], 3.0, rtol=1e-15)


def test_exact_rule_equals_reference_where_no_chunk_repeats():
    # the two rules only differ when groups of one chunk merge the same
    # class set; on full grids (n = m^k) and at m = n they agree
    rng = np.random.default_rng(3)
    for n, m in [(4, 2), (8, 2), (9, 3), (16, 4), (27, 3), (7, 7), (13, 13)]:
        vals = rng.standard_normal((n, 3))
        _same_result(sp.run_plan(n, m, vals, exact=True), ref.run_plan(n, m, vals))


def test_weighted_butterfly_m_equals_n_reference_known_answers():
    # SPEC.md:219-221, 246 through the reference's own executor
    assert (ref.run_plan(9, 3, np.arange(1.0, 10.0).reshape(9, 1))["values"] == 5.0).all()
    assert (ref.run_plan(4, 2, np.array([[0.0], [0.0], [0.0], [4.0]]))["values"] == 1.0).all()
    rng = np.random.default_rng(9)
    rows = [rng.standard_normal(1000).astype(np.float32) for _ in range(6)]
    w = [3.0, 0.0, 1.0, 2.0, 5.0, 1.0]
    mean = ref.weighted_mean(rows, w, block=256)
    res = ref.run_plan(6, 6, np.stack(rows).astype(np.float64), w)
    np.testing.assert_array_equal(mean, res["values"][0])


# --------------------------------------------------------------- model.cpp
def _mutations(base: dict):
    """Specs derived from `base`: every check of validate() and every
    SpecParseError path of spec_from_json (model.cpp:38-146)."""
    out = []

    def mut(f):
        s = copy.deepcopy(base)
        f(s)
        out.append(json.dumps(s))

    for key, vals in [("batch_size", [0.0, -1.0, "x", None]), ("param_count", [0.0, -5.0, "y"]),
                      ("bits_per_param", [0.0, -16.0, True])]:
        for v in vals:
            mut(lambda s, k=key, v=v: s.__setitem__(k, v))
    mut(lambda s: s.pop("param_count"))
    mut(lambda s: s.pop("peers"))
    mut(lambda s: s.__setitem__("peers", {}))
    mut(lambda s: s.__setitem__("peers", []))
    for field, vals in [("samples_per_sec", [-1.0, "a", 0.0]), ("download_mbps", [0.0, -3.0, "b", None]),
                        ("upload_mbps", [0.0, "c"]), ("failure_rate", [1.0, -0.1, 0.5]),
                        ("can_compute", [False, 1]), ("client_mode", [True, "no"]), ("id", ["", 7])]:
        for v in vals:
            mut(lambda s, f=field, v=v: s["peers"][1].__setitem__(f, v))
    for field in ("id", "download_mbps", "upload_mbps"):
        mut(lambda s, f=field: s["peers"][0].pop(f))
    mut(lambda s: s["peers"][1].__setitem__("id", s["peers"][0]["id"]))
    mut(lambda s: [p.__setitem__("can_compute", False) for p in s["peers"]])
    mut(lambda s: s["peers"][0].update(can_compute=False))
    ids = [p["id"] for p in base["peers"]]
    for link in [{"from": ids[0], "to": ids[1], "mbps": 20.0}, {"from": ids[0], "to": ids[0], "mbps": 1.0},
                 {"from": ids[0], "to": ids[1], "mbps": -1.0}, {"from": ids[0], "to": "ghost", "mbps": 1.0},
                 {"from": ids[0], "to": ids[1]}, {"from": ids[0], "mbps": 3.0},
                 {"from": ids[1], "to": ids[0], "mbps": "fast"}]:
        mut(lambda s, l=link: s.__setitem__("links", [l]))
    for text in ["{not json", "[]", "3", '{"peers": []}', '{"param_count": 1}',
                 '{"param_count": 1, "peers": [{"id": "a"}]}']:
        out.append(text)
    return out


def _corpus():
    specs = [json.dumps(homogeneous(3, mbps=250.0))]
    specs += [spec_json(name) for name in sorted(FLEETS)]
    if os.path.isdir(SCENARIOS):
        for f in sorted(os.listdir(SCENARIOS)):
            text = open(os.path.join(SCENARIOS, f)).read()
            try:
                sc = json.loads(text)
            except ValueError:  # bad.json: a parse-error fixture
                specs.append(text)
                continue
            if "collaboration" in sc:
                specs.append(json.dumps(sc["collaboration"]))
    base = homogeneous(3, mbps=250.0)
    base["peers"][2]["client_mode"] = True
    return specs + _mutations(base)


def _ours_validate(text):
    return [(v["peer"], v["field"], v["message"]) for v in sp.validate_spec(text)]


def test_validate_and_parse_errors_match_reference():
    n_err = n_viol = 0
    for text in _corpus():
        try:
            want = ref.validate(text)
        except ValueError as e:
            n_err += 1
            with pytest.raises(ValueError) as got:
                sp.validate_spec(text)
            assert str(got.value) == str(e), text
            continue
        n_viol += bool(want)
        assert _ours_validate(text) == want, text
    assert n_err >= 10 and n_viol >= 15  # the corpus reaches both paths


def test_spec_json_round_trip_matches_reference():
    for text in _corpus():
        try:
            want = ref.spec_roundtrip(text)
        except ValueError:
            continue
        assert sp.spec_roundtrip(text) == want


@pytest.mark.parametrize("name", ["homogeneous8", "het8c", "het4b", "aux_server"])
def test_assignment_json_matches_reference(name):
    text = spec_json(name)
    d = sp.solve_strategy(text)
    want = ref.assignment_json(text, d["gradient_flows"], d["average_flows"], d["duty_cycle"],
                               d["compute"], d["fractions"], d["steps_per_sec"], d["lp_iterations"])
    assert sp.assignment_json(text) == want
