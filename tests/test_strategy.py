"""Strategy optimizer (host C++ LP) vs the reference's goldens.

Ports /root/reference/proj/tests/cpp/test_strategy.cpp to the Python binding,
plus the unique-fraction fixtures of SURVEY.md Appendix A (HiGHS-probed) and
scipy HiGHS as a second, independent oracle for xi (oracle/lp_highs.py)."""
import json
import math
import time

import numpy as np
import pytest

from golden.fleets import (FLEETS, FRACTIONS_APPENDIX_A, XI_APPENDIX_A, XI_GOLDEN, homogeneous,
                           spec_json)
from paper_2106_10207_b200 import _swarmplan as sp


def _sj(d):
    return json.dumps(d)


def check_assignment(spec, s):
    """test_strategy.cpp:48-84: the optimizer's own head-room identities."""
    n = len(spec["peers"])
    P = spec["param_count"] * spec.get("bits_per_param", 32.0)
    cap = max([1.0] + [max(p["download_mbps"], p["upload_mbps"]) * 1e6 for p in spec["peers"]])
    slack = 1e-6 * max(P, cap)
    supply = sum(p["samples_per_sec"] * c for p, c in zip(spec["peers"], s["duty_cycle"]))
    assert s["steps_per_sec"] <= supply / spec["batch_size"] + 1e-6
    a, g = np.array(s["gradient_flows"]), np.array(s["average_flows"])
    for i, p in enumerate(spec["peers"]):
        if p.get("can_compute", True) and not p.get("client_mode", False):
            assert g[:, i].sum() >= s["steps_per_sec"] * P - slack
    for i, p in enumerate(spec["peers"]):
        inflow = sum(a[j, i] + g[j, i] for j in range(n) if j != i)
        outflow = sum(a[i, j] + g[i, j] for j in range(n) if j != i)
        assert inflow <= p["download_mbps"] * 1e6 + slack
        assert outflow <= p["upload_mbps"] * 1e6 + slack
        assert s["fractions"][i] >= 0.0
    assert math.isclose(sum(s["fractions"]), 1.0, rel_tol=1e-9)


# ------------------------------------------------------------- LP shape
def test_reference_program_shape_two_peers():
    spec = homogeneous(2, 1.0, 100.0, 2.0, 1e6)
    spec["links"] = [{"from": "peer0", "to": "peer1", "mbps": 20.0},
                     {"from": "peer1", "to": "peer0", "mbps": 30.0}]
    sh = sp.build_lp_shape(_sj(spec))
    assert sh["num_vars"] == 2 * 4 + 2 + 1
    assert (sh["rows_compute"], sh["rows_aggregate"], sh["rows_service"]) == (1, 2, 8)
    assert (sh["rows_download"], sh["rows_upload"], sh["rows_link"]) == (2, 2, 2)
    assert sh["rows"] == 1 + 2 + 8 + 2 + 2 + 2


def test_non_computing_peers_excluded_from_compute_families():
    spec = homogeneous(3, 1.0, 100.0, 2.0, 1e6)
    spec["peers"][2].update(samples_per_sec=0.0, can_compute=False)
    sh = sp.build_lp_shape(_sj(spec))
    assert sh["rows_service"] == 9 * 2
    assert sh["rows_aggregate"] == 2


def test_client_mode_rows():
    spec = homogeneous(3, 1.0, 100.0, 2.0, 1e6)
    spec["peers"][1]["client_mode"] = True
    assert sp.build_lp_shape(_sj(spec))["rows_aggregate"] == 2


# -------------------------------------------------------------- goldens
def test_single_peer_runs_at_own_rate():
    s = sp.solve_strategy(_sj(homogeneous(1, 2.0, 100.0, 4.0, 1e6)))
    assert s["steps_per_sec"] == pytest.approx(0.5)
    assert s["compute"][0] and s["duty_cycle"][0] == pytest.approx(1.0)


def test_homogeneous_fleet_splits_evenly():
    s = sp.solve_strategy(spec_json("homogeneous8"))
    assert s["steps_per_sec"] == pytest.approx(0.697544642857, rel=1e-9)
    assert all(s["compute"])
    for f in s["fractions"]:
        assert f == pytest.approx(0.125, rel=1e-6)
    check_assignment(json.loads(spec_json("homogeneous8")), s)


def test_well_connected_helper_absorbs_all_aggregation():
    s = sp.solve_strategy(spec_json("aux_server"))
    assert s["steps_per_sec"] == pytest.approx(1.220703125, rel=1e-9)
    assert s["fractions"][8] == pytest.approx(1.0, rel=1e-6)
    check_assignment(json.loads(spec_json("aux_server")), s)


@pytest.mark.parametrize("name", ["table1_a", "table1_b", "table1_c", "table1_d", "daynight",
                                  "static16"])
def test_frozen_xi_goldens(name):
    s = sp.solve_strategy(spec_json(name))
    assert s["steps_per_sec"] == pytest.approx(XI_GOLDEN[name], rel=1e-9)
    check_assignment(json.loads(spec_json(name)), s)


@pytest.mark.parametrize("name", ["het8c", "het4b"])
def test_unique_fraction_fixtures(name):
    s = sp.solve_strategy(spec_json(name))
    assert s["steps_per_sec"] == pytest.approx(XI_APPENDIX_A[name], rel=1e-9)
    np.testing.assert_allclose(s["fractions"], FRACTIONS_APPENDIX_A[name], atol=1e-6)
    check_assignment(json.loads(spec_json(name)), s)


def test_table1_d_concentrates_aggregation_on_fast_peer():
    # SPEC.md:543 "aggregator role concentrated on the 2.5 Gb/s peer"
    s = sp.solve_strategy(spec_json("table1_d"))
    assert max(range(17), key=lambda i: s["fractions"][i]) == 16
    assert s["fractions"][16] > 0.8


def _random_small_spec(seed):
    rng = np.random.default_rng(seed)
    n = 2 + int(rng.integers(0, 2))
    spec = {"batch_size": float(1 + 3 * rng.uniform()), "param_count": float(1e6 + 4e6 * rng.uniform()),
            "peers": []}
    for i in range(n):
        spec["peers"].append({"id": f"p{i}", "samples_per_sec": float(0.5 + 2.5 * rng.uniform()),
                              "download_mbps": float(10 + 190 * rng.uniform()),
                              "upload_mbps": float(10 + 190 * rng.uniform())})
    if rng.uniform() < 0.25:
        spec["peers"][-1]["client_mode"] = True
    return spec


@pytest.mark.parametrize("seed", range(1, 31))
def test_random_fleets_satisfy_own_constraints(seed):
    spec = _random_small_spec(seed)
    s = sp.solve_strategy(_sj(spec))
    check_assignment(spec, s)
    assert s["lp_iterations"] > 0


@pytest.mark.parametrize("seed", range(50, 81))
def test_binary_masks_never_beat_relaxation(seed):
    """test_strategy.cpp:240-259: relaxed LP >= best 0/1 mask == shipped xi."""
    spec = _random_small_spec(seed)
    sj = _sj(spec)
    n = len(spec["peers"])
    best = 0.0
    for mask in range(1, 1 << n):
        st, xi = sp.reference_program_xi(sj, [(mask >> b) & 1 for b in range(n)])
        if st == "optimal":
            best = max(best, xi)
    st, relaxed = sp.reference_program_xi(sj, [])
    assert st == "optimal"
    assert relaxed >= best - 1e-6 * max(1.0, best)
    shipped = sp.solve_strategy(sj)["steps_per_sec"]
    assert shipped == pytest.approx(best, rel=1e-6)
    assert shipped <= relaxed + 1e-6 * max(1.0, relaxed)


@pytest.mark.parametrize("n", range(2, 7))
def test_idle_helper_never_slows_fleet(n):
    spec = homogeneous(n, 1.0, 100.0, float(n), 2e6)
    base = sp.solve_strategy(_sj(spec))["steps_per_sec"]
    spec["peers"].append({"id": "helper", "samples_per_sec": 0.0, "download_mbps": 400.0,
                          "upload_mbps": 400.0, "can_compute": True})
    assert sp.solve_strategy(_sj(spec))["steps_per_sec"] >= base - 1e-9


def test_client_peers_compute_but_never_aggregate():
    spec = homogeneous(4, 1.0, 100.0, 4.0, 2e6)
    spec["peers"][3]["client_mode"] = True
    s = sp.solve_strategy(_sj(spec))
    assert s["fractions"][3] == pytest.approx(0.0, abs=1e-12)
    a, g = np.array(s["gradient_flows"]), np.array(s["average_flows"])
    for j in range(3):
        assert a[j, 3] == pytest.approx(0.0, abs=1e-6) and g[j, 3] == pytest.approx(0.0, abs=1e-6)
    assert s["duty_cycle"][3] > 0.0
    check_assignment(spec, s)


# ---------------------------------------------------------- round models
def test_allreduce_round_model():
    spec = homogeneous(4, 1.0, 100.0, 4.0, 25e6)
    spec["peers"][2]["upload_mbps"] = 50.0
    P = 25e6 * 32
    assert sp.simulate_averaging(_sj(spec), "allreduce") == pytest.approx(2 * 0.75 * P / 50e6)
    spec["links"] = [{"from": "peer0", "to": "peer1", "mbps": 10.0}]
    assert sp.simulate_averaging(_sj(spec), "allreduce") == pytest.approx(2 * 0.75 * P / 10e6)
    assert sp.simulate_averaging(_sj(homogeneous(1, 1.0, 100.0, 1.0, 25e6)), "allreduce") == 0.0


def test_parameter_server_round_model():
    spec = homogeneous(4, 1.0, 100.0, 4.0, 25e6)
    spec["peers"][0].update(download_mbps=400.0, upload_mbps=300.0)
    P = 25e6 * 32
    assert sp.simulate_averaging(_sj(spec), "parameter_server", 0) == pytest.approx(3 * P / 300e6)
    assert sp.simulate_averaging(_sj(spec), "ps", 1) == pytest.approx(3 * P / 100e6)
    with pytest.raises(ValueError):
        sp.simulate_averaging(_sj(spec), "parameter_server", 7)


def test_adaptive_round_two_peer_closed_form():
    """test_strategy.cpp:318-325 expects P / (2 * 100e6), but the reference's
    own communication-only program (strategy.cpp:193-295 with c pinned to 1)
    has optimum P / 100e6: each peer uploads its gradient half AND the
    averaged half over one 100 Mbit/s uplink. scipy HiGHS on the same program
    (oracle/lp_highs.py) agrees with P / 100e6, so that is the value pinned
    here ('reference test inconsistencies')."""
    from oracle import lp_highs

    spec = homogeneous(2, 1.0, 100.0, 2.0, 25e6)
    P = 25e6 * 32
    t = sp.simulate_averaging(_sj(spec), "adaptive")
    assert t == pytest.approx(P / 100e6, rel=1e-6)
    comm_only = homogeneous(2, 1e9, 100.0, 2.0, 25e6)  # compute row never binds
    assert 1.0 / lp_highs.solve(comm_only)[0] == pytest.approx(t, rel=1e-9)


def test_invalid_specs_rejected():
    spec = homogeneous(2, 1.0, 100.0, 2.0, 1e6)
    spec["batch_size"] = 0.0
    with pytest.raises(ValueError):
        sp.solve_strategy(_sj(spec))
    with pytest.raises(ValueError):
        sp.build_lp_shape(_sj(spec))


def test_repeat_solves_bit_identical():
    a = sp.solve_strategy(spec_json("aux_server"))
    b = sp.solve_strategy(spec_json("aux_server"))
    assert a == b


def test_compare_strategies_ordering_setup_c():
    rows = {r["algorithm"]: r for r in sp.compare_strategies(spec_json("table1_c"))}
    # PAPER.md:238 (Table 1, setup C): DeDLOC beats all-reduce and PS
    assert rows["adaptive"]["round_s"] < rows["allreduce"]["round_s"] < rows["parameter_server"]["round_s"]
    assert rows["allreduce"]["round_s"] / rows["adaptive"]["round_s"] == pytest.approx(1.917, rel=0.01)


def test_plan_parts_feeds_the_round():
    d = sp.plan_parts(spec_json("het8c"), 17847474, 8)
    offs = d["offsets"]
    assert offs[0] == 0 and offs[-1] == 17847474
    lens = np.diff(offs)
    assert lens[6] == 0
    assert abs(lens[7] / 17847474 - 0.7) < 1e-5
    assert sp.part_offsets(17847474, d["fractions"], 8) == offs


def test_solve_time_n8_budget():
    # the paper's solver budget is < 50 ms; n = 8 is the GPU
    # fleet size of this framework
    t0 = time.perf_counter()
    sp.solve_strategy(spec_json("homogeneous8"))
    assert time.perf_counter() - t0 < 0.5


@pytest.mark.parametrize("name", ["homogeneous8", "aux_server", "table1_b", "table1_d", "static16",
                                  "het8c", "het4b"])
def test_highs_oracle_agrees(name):
    """scipy HiGHS restatement of Eq. 5 (oracle/lp_highs.py) reproduces the
    reference goldens, and our solver matches it."""
    from oracle import lp_highs

    xi_h, fr_h = lp_highs.solve(json.loads(spec_json(name)))
    gold = XI_GOLDEN.get(name, XI_APPENDIX_A.get(name))
    assert xi_h == pytest.approx(gold, rel=1e-9)
    s = sp.solve_strategy(spec_json(name))
    assert s["steps_per_sec"] == pytest.approx(xi_h, rel=1e-9)
    if name in FRACTIONS_APPENDIX_A or name in ("homogeneous8", "aux_server"):
        np.testing.assert_allclose(s["fractions"], fr_h, atol=1e-6)


def test_compare_strategies_with_measured_round_times():
    # executor round times replace the fluid model's comm time
    sj = spec_json("het4b")
    model = {r["algorithm"]: r for r in sp.compare_strategies(sj)}
    meas = {"allreduce": 2e-4, "parameter_server": 5e-4, "adaptive": 1e-4}
    rows = {r["algorithm"]: r for r in sp.compare_strategies(sj, meas)}
    spec = json.loads(sj)
    compute_s = spec["batch_size"] / sum(p["samples_per_sec"] for p in spec["peers"])
    for alg, sec in meas.items():
        assert rows[alg]["round_s"] == sec
        if alg != "adaptive":  # adaptive's compute uses duty-cycled rates
            assert rows[alg]["steps_per_hour"] == pytest.approx(3600.0 / max(compute_s, sec))
    # a partial map keeps the model for the rest
    part = {r["algorithm"]: r for r in sp.compare_strategies(sj, {"adaptive": 1e-4})}
    assert part["allreduce"] == model["allreduce"]
    with pytest.raises(ValueError):
        sp.compare_strategies(sj, {"gossip": 1.0})
    with pytest.raises(ValueError):
        sp.compare_strategies(sj, {"adaptive": -1.0})


def test_measured_fractions_per_algorithm():
    from paper_2106_10207_b200.measure import fractions_for

    sj = spec_json("het4b")
    assert fractions_for(sj, "allreduce") == [0.25] * 4
    assert fractions_for(sj, "parameter_server") == [0.0, 0.0, 0.0, 1.0]
    np.testing.assert_allclose(fractions_for(sj, "adaptive"), [1 / 22] * 3 + [19 / 22], atol=1e-9)


@pytest.mark.parametrize("n", [2, 3, 5, 6])
def test_symmetric_fleets_get_symmetric_fractions(n):
    # the LP optimum of a homogeneous fleet is not unique for every n (two
    # peers: [1, 0] and [0.5, 0.5] tie); solve_strategy returns the average
    # over interchangeable peers, which keeps every stage optimal
    spec = homogeneous(n, 1.0, 1000.0, 4096.0, 17847474)
    s = sp.solve_strategy(_sj(spec))
    np.testing.assert_allclose(s["fractions"], [1.0 / n] * n, rtol=1e-12)
    check_assignment(spec, s)


@pytest.mark.parametrize("name", ["table1_c", "daynight", "table1_d", "aux_server"])
def test_symmetrized_assignment_feasible(name):
    spec = json.loads(spec_json(name))
    s = sp.solve_strategy(spec_json(name))
    check_assignment(spec, s)
    assert s["steps_per_sec"] == pytest.approx(XI_GOLDEN[name], rel=1e-9)
    # interchangeable peers (same spec and duty cycle) get equal fractions
    groups = {}
    for p, f, c in zip(spec["peers"], s["fractions"], s["duty_cycle"]):
        key = (p["samples_per_sec"], p["download_mbps"], p["upload_mbps"],
               p.get("can_compute", True), p.get("client_mode", False), round(c, 9))
        groups.setdefault(key, []).append(f)
    for fs in groups.values():
        assert max(fs) - min(fs) <= 1e-12
