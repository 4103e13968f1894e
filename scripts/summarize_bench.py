#!/usr/bin/env python
"""Markdown table of bench.py lines (one JSON object per file), with the
round roofline recomputed by bench.py's current model so lines measured
under an older model compare on the same footing."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2106_10207_b200 import fleets  # noqa: E402
from paper_2106_10207_b200.dist import plan_round  # noqa: E402


def main(paths):
    print("| file | N | workload | LAMB | round (us) | GB/s | T_roof (us) | frac | e2e GB/s |")
    print("|---|---|---|---|---|---|---|---|---|")
    for path in paths:
        lines = [ln for ln in open(path) if ln.startswith("{")]
        if not lines:
            continue
        d = json.loads(lines[-1])
        if d.get("impl") == "reference" or "config" not in d or "peers_per_gpu" not in d["config"]:
            continue
        c = d["config"]
        n, world, L, wire = c["params"], d["n_gpus"], c["peers_per_gpu"], c["wire"]
        G = world * L
        blk = c.get("q8_block") or 4096
        shard = c.get("lamb", "replicated").startswith("sharded")
        fused = not shard and d["kernel_ms"]["update_ms"] < 0.1 * d["kernel_ms"]["moments_ms"]
        wl = c["workload"].split(":")[0]
        fleet = bench.WORKLOADS.get(wl, (None, None, None, None))[3]
        sj = fleets.spec_json(fleet) if fleet else json.dumps(fleets.homogeneous(G, 1.0, 1000.0, 4096.0, n))
        offs = plan_round(sj, n, blk if wire == "q8" else 8)["offsets"]
        b = bench.wire_bytes(wire, blk)
        ms = [bench.rank_model(r, offs, L, world, n, b, wire, shard, fused,
                               world == 1 and L == 1 and wire != "q8" and fused) for r in range(world)]
        t = bench.overlap_roofline(ms, n, 6524.0) * 1e6
        e2e = (d.get("e2e") or {}).get("value")
        print(f"| {os.path.basename(path)} | {world} | {wl} | {'sharded' if shard else 'replicated'} | "
              f"{d['round_us']:.1f} | {d['value']:.0f} | {t:.1f} | {t / d['round_us']:.3f} | {e2e} |")


if __name__ == "__main__":
    main(sys.argv[1:])
