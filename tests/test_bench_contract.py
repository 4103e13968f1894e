"""bench.py's contract on CPU: the reference arm prints exactly one JSON line
with the keys the driver reads, the fleet workloads plan through the LP, and
the sweep tensor table covers the requested size (the GPU arm is exercised
on the B200 box)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _ref(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", *args],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout  # one JSON line, nothing else on stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("args", [("--workload", "het4b-fp32"),
                                  ("--workload", "sweep", "--params", "1000003", "--wire", "q8")])
def test_reference_arm_line(args):
    d = _ref(*args)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "impl", "cpu_baseline", "e2e", "config"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # the reference's own run_plan (oracle/_ref) carries the averaging
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert set(d["phase_ms"]) == {"pack_ms", "average_ms", "to_wire_ms", "lamb_ms"}


def test_sweep_tensor_table():
    import bench

    t = bench.tensor_table("uniform4m", 1 << 30)
    assert sum(t) == 1 << 30 and max(t) == 4 << 20
    t = bench.tensor_table("uniform4m", 10_000_001)
    assert sum(t) == 10_000_001 and t[-1] == 10_000_001 % (4 << 20)
    with pytest.raises(SystemExit):
        bench.tensor_table("uniform4m", 0)


def test_fleet_workloads_plan_through_the_lp():
    import bench
    from paper_2106_10207_b200 import fleets
    from paper_2106_10207_b200.dist import plan_round

    for name, (table, wire, block, fleet) in bench.WORKLOADS.items():
        if fleet is None:
            continue
        n = sum(bench.tensor_table(table))
        plan = plan_round(fleets.spec_json(fleet), n, block if wire == "q8" else 8)
        G = len(json.loads(fleets.spec_json(fleet))["peers"])
        assert len(plan["offsets"]) == G + 1 and plan["offsets"][-1] == n
        assert all(w > 0 for w in plan["weights"])
