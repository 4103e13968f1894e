"""Collaboration specs of the reference's scenarios, written as peer-group tables.

The reference fixtures (/root/reference/proj/scenarios/*.json) are uniform
groups of peers; each entry below names the file it restates and lists
(count, samples_per_sec, download_mbps, upload_mbps, extra flags). het8c /
het4b are the unique-fraction fixtures of SURVEY.md Appendix A (BASELINE
configs 4 and 1). bench.py plans its rounds from these through the LP
(solve_strategy -> part_offsets); tests/golden/fleets.py adds the goldens."""
import json

FLEETS = {
    # name: (batch_size, param_count, [(count, s, d, u, flags)], source)
    "homogeneous8": (8.0, 25.6e6, [(8, 1.0, 1000.0, 1000.0, {})], "scenarios/homogeneous8.json"),
    "table1_a": (8.0, 25.6e6, [(8, 1.0, 1000.0, 1000.0, {})], "scenarios/table1_a.json"),
    "table1_b": (1.0, 25.6e6, [(16, 1.0, 200.0, 200.0, {})], "scenarios/table1_b.json"),
    "table1_c": (1.0, 25.6e6, [(8, 1.0, 1000.0, 1000.0, {}), (16, 1.0, 200.0, 200.0, {})],
                 "scenarios/table1_c.json"),
    "table1_d": (1.0, 25.6e6, [(16, 1.0, 200.0, 200.0, {}), (1, 1.0, 2500.0, 2500.0, {})],
                 "scenarios/table1_d.json"),
    "daynight": (8.0, 1e6, [(24, 1.0, 1000.0, 1000.0, {})], "scenarios/daynight.json"),
    "static16": (8.0, 1e6, [(16, 1.0, 1000.0, 1000.0, {})], "scenarios/static16.json"),
    "aux_server": (4.0, 25.6e6, [(8, 1.0, 1000.0, 1000.0, {}),
                                 (1, 0.0, 100000.0, 100000.0, {"can_compute": False})],
                   "scenarios/aux_server.json"),
    "no_compute": (1.0, 25.6e6, [(4, 0.0, 1000.0, 1000.0, {"can_compute": False})],
                   "scenarios/no_compute.json"),
    # SURVEY.md Appendix A (unique fractions; HiGHS DS = IPM)
    "het8c": (8.0, 17847474.0, [(6, 1.0, 200.0, 200.0, {}), (1, 1.0, 200.0, 200.0, {"client_mode": True}),
                                (1, 1.0, 800.0, 800.0, {})], "SURVEY.md Appendix A"),
    "het4b": (4.0, 11813810.0, [(3, 1.0, 200.0, 200.0, {}), (1, 1.0, 500.0, 500.0, {})],
              "SURVEY.md Appendix A"),
}


def spec(name: str) -> dict:
    batch, params, groups, _ = FLEETS[name]
    peers = []
    for count, s, d, u, flags in groups:
        for _ in range(count):
            p = {"id": f"peer{len(peers)}", "samples_per_sec": s, "download_mbps": d,
                 "upload_mbps": u}
            p.update(flags)
            peers.append(p)
    return {"peers": peers, "batch_size": batch, "param_count": params, "bits_per_param": 32.0}


def spec_json(name: str) -> str:
    return json.dumps(spec(name))


def homogeneous(n, samples=1.0, mbps=1000.0, batch=1.0, params=1e6):
    return {"peers": [{"id": f"peer{i}", "samples_per_sec": samples, "download_mbps": mbps,
                       "upload_mbps": mbps} for i in range(n)],
            "batch_size": batch, "param_count": params, "bits_per_param": 32.0}
