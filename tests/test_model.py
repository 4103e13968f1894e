"""Spec validation and JSON (swarmplan model) — ports of
/root/reference/proj/tests/cpp/test_model.cpp and tests/python/test_smoke.py."""
import json

import pytest

from golden.fleets import homogeneous
from paper_2106_10207_b200 import _swarmplan as sp


def test_valid_spec_has_no_violations():
    assert sp.validate_spec(json.dumps(homogeneous(2))) == []


def test_violation_order_and_fields():
    spec = homogeneous(3)
    spec["batch_size"] = 0.0
    spec["peers"][0]["download_mbps"] = -1.0
    spec["peers"][1]["can_compute"] = False  # but samples_per_sec = 1
    spec["peers"][2]["failure_rate"] = 1.0
    v = sp.validate_spec(json.dumps(spec))
    assert v[0]["peer"] == -1 and v[0]["field"] == "batch_size"
    assert [(x["peer"], x["field"]) for x in v[1:]] == [
        (0, "download_bps"), (1, "samples_per_sec"), (2, "failure_rate")]


def test_duplicate_ids_and_links():
    spec = homogeneous(2)
    spec["peers"][1]["id"] = "peer0"
    assert any(x["field"] == "id" for x in sp.validate_spec(json.dumps(spec)))
    spec = homogeneous(2)
    spec["links"] = [{"from": "peer0", "to": "peer0", "mbps": 5.0}]
    assert any(x["field"] == "links" for x in sp.validate_spec(json.dumps(spec)))
    spec["links"] = [{"from": "peer0", "to": "nobody", "mbps": 5.0}]
    with pytest.raises(sp.SpecParseError):
        sp.validate_spec(json.dumps(spec))


def test_no_compute_fleet_rejected():
    spec = homogeneous(4, samples=0.0)
    for p in spec["peers"]:
        p["can_compute"] = False
    assert any(x["message"] == "no peer contributes compute throughput"
               for x in sp.validate_spec(json.dumps(spec)))
    with pytest.raises(ValueError):
        sp.solve_strategy(json.dumps(spec))


@pytest.mark.parametrize("text", ["{not json", "[]", '{"peers": []}', '{"param_count": 1}',
                                  '{"param_count": 1, "peers": [{"id": "a"}]}',
                                  '{"param_count": 1, "peers": [{"id": "a", "download_mbps": "x", "upload_mbps": 1}]}'])
def test_parse_errors_are_value_errors(text):
    with pytest.raises(ValueError):
        sp.solve_strategy(text)


def test_spec_round_trip_through_scenario():
    spec = homogeneous(3, mbps=250.0)
    spec["peers"][2]["client_mode"] = True
    spec["links"] = [{"from": "peer0", "to": "peer1", "mbps": 20.0}]
    out = json.loads(sp.scenario_spec_json(json.dumps({"name": "x", "collaboration": spec})))
    assert out["peers"][2]["client_mode"] is True
    assert out["peers"][0]["download_mbps"] == 250.0
    assert out["links"] == [{"from": "peer0", "to": "peer1", "mbps": 20.0}]


def test_assignment_json_shape():
    a = json.loads(sp.assignment_json(json.dumps(homogeneous(4))))
    assert list(a) == ["steps_per_sec", "lp_iterations", "peers", "gradient_flow_bps",
                       "partition_flow_bps"]
    assert [p["aggregation_fraction"] for p in a["peers"]] == pytest.approx([0.25] * 4)


# -- tests/python/test_smoke.py of the reference, against the drop-in package
def test_reference_python_smoke():
    import swarmplan

    spec = json.dumps(homogeneous(4, mbps=1000.0))
    out = swarmplan.solve_strategy(spec)
    assert out["steps_per_sec"] > 0 and all(out["compute"])
    assert sum(out["fractions"]) == pytest.approx(1.0, rel=1e-6)
    for f in out["fractions"]:
        assert f == pytest.approx(0.25, abs=1e-6)
    ar = swarmplan.simulate_averaging(json.dumps(homogeneous(8)), "allreduce")
    ps = swarmplan.simulate_averaging(json.dumps(homogeneous(8)), "parameter_server")
    assert ar > 0 and ps > ar
    assert len(swarmplan.build_plan(16, 4)) == 2
    assert swarmplan.optimal_group_size(16, 0.0) == 16
    assert swarmplan.expected_iterations(16, 16, 0.0) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        swarmplan.solve_strategy("{not json")
    with pytest.raises(NotImplementedError):
        swarmplan.run_training("{}", hours=0.25)  # churn simulation: out of scope
