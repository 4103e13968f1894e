#!/usr/bin/env python
"""Markdown table of sweep lines (scripts/sweep.py output), with the round
roofline recomputed by bench.py's current phase model (so lines measured
under an older model compare on the same footing)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main(paths):
    print("| N | params | wire | LAMB | round (us) | GB/s | T_roof (us) | frac | T serialized §8d (us) | frac |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for path in paths:
        for line in open(path):
            d = json.loads(line)
            if "error" in d:
                print(f"| {d['n_gpus']} | {d['params']} | {d['wire']} | | error | | | | | |")
                continue
            c = d["config"]
            n, world, L, wire = c["params"], d["n_gpus"], c["peers_per_gpu"], c["wire"]
            G = world * L
            shard = c["lamb"].startswith("sharded")
            fused = not shard and d["kernel_ms"]["update_ms"] < 0.1 * d["kernel_ms"]["moments_ms"]
            offs = [round(i * n / G / 8) * 8 for i in range(G)] + [n]
            b = bench.wire_bytes(wire, c["q8_block"] or 4096)
            if wire == "q8":
                blk = c["q8_block"]
                offs = [round(i * n / G / blk) * blk for i in range(G)] + [n]
            ms = [bench.rank_model(r, offs, L, world, n, b, wire, shard, fused,
                                   world == 1 and L == 1 and wire != "q8" and fused)
                  for r in range(world)]
            peak = 6524.0
            t = bench.round_roofline(ms, n, peak) * 1e6
            t2 = bench.overlap_roofline(ms, n, peak) * 1e6
            print(f"| {world} | {n:,} | {wire} | {'sharded' if shard else 'replicated'} | "
                  f"{d['round_us']:.1f} | {d['value']:.0f} | {t2:.1f} | {t2 / d['round_us']:.3f} | "
                  f"{t:.1f} | {t / d['round_us']:.3f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
