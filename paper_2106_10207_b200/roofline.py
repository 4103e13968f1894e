"""Byte model and roofline of the averaging round.

Per rank r owning the fraction f of the vector (from the LP offsets), with
L local peers, `world` ranks and wire width b bytes, the round moves:
  pack + scatter : HBM 4 L + G f b; NVLink max(L (1 - f) b out, (G - L) f b in)
  reduce         : HBM G f b + (f b sharded | b replicated); NVLink (replicated)
                   max((world - 1) f b out, (1 - f) b in)
  LAMB           : HBM f_l (24 + b) (+ (1 - f) 4 received parameters, sharded);
                   NVLink (sharded) max((world - 1) f 4 out, (1 - f) 4 in)
where f_l = f when sharded, 1 when replicated. The phases are separated by
cross-rank barriers, so a lower bound on the round time is the sum over
phases of the slowest rank's max(HBM time, NVLink time) (`overlap_roofline`).
Denominators: HBM 6524 GB/s measured copy (MEASURED_PEAKS.json), NVLink
770 GB/s measured peer copy per direction (B200_PROFILING.md; 900 nominal).
`choose_shard_lamb` picks the LAMB mode with the lower bound for a plan.
"""
from __future__ import annotations

NVLINK_GBS = 770.0
HBM_GBS = 6524.0
# Sharded rounds run ~10 % further from their bound than replicated ones
# (measured on 2 and 4 B200s, profiles/r01/lamb_mode.txt: the parameter push
# moves 9-18 MB per pair, below the link's large-copy rate)
SHARD_PENALTY = 1.1


def rank_model(r, offsets, L, world, n, b, wire, shard, fused_pack) -> dict:
    """Algorithmic bytes for rank r given the part fraction f
    it owns.

    `alg`: per-kernel §8(d) bytes of one launch (pack 4 + b per packed
    element, weighted reduce G f b + f b, LAMB 24 + b per stepped element;
    one GPU with one peer runs the pack inside LAMB, so k_lamb's launch
    carries both: 28 + 2b). `impl`: the bytes k_lamb actually moves through
    L2 per launch: §8(d)'s LAMB bytes plus pass 2's re-read of p (4 B; u
    comes from the shared-memory stash), and with the fused pack its fp32
    read and wire store (4 + b) but no wire re-read.
    `phases`: for each phase of the round (pack+scatter, reduce(+push),
    LAMB(+parameter push)) the HBM bytes and the NVLink bytes per direction
    (the larger of out and in), per element of the vector. Phases are
    separated by cross-rank barriers, so the round's roofline is the sum over
    phases of the slowest rank's max(HBM time, NVLink time)."""
    G = L * world
    f = (offsets[(r + 1) * L] - offsets[r * L]) / n
    f_l = f if shard else 1.0  # fraction of the vector this rank's LAMB steps
    pack_alg = 0.0 if (fused_pack or (wire == "fp32" and world == 1)) else L * n * (4 + b)
    alg = {
        "pack_ms": pack_alg,
        "reduce_ms": (G * f * b + f * b) * n if G > 1 else 0.0,
        "lamb_ms": f_l * n * (24 + b) + (n * (4 + b) if fused_pack else 0.0),
    }
    impl = {"lamb_ms": f_l * n * (24 + b + 4) + (n * 4.0 if fused_pack else 0.0)}
    multi = world > 1
    # pack: read the fp32 gradients (4 L), write the wire of the owned range
    # (L f b from local peers, (G - L) f b arriving from the other ranks; the
    # rest of the local wire lands in the owners' HBM). fp32 on one GPU: the
    # wire is the gradient itself (zero-copy).
    pack_hbm = (4 * L + G * f * b) if (wire != "fp32" or multi) else 0.0
    pack_nvl = max(L * (1 - f) * b, (G - L) * f * b) if multi else 0.0
    # reduce: read G inbox slots of the owned range, write the average
    # (replicated: pushed to every rank, (1 - f) b arrives from the others).
    # G = 1: the average of one peer is its wire values, no reduce pass.
    if G > 1:
        # sharded: the average stays local (f b); replicated: f b written
        # here and pushed out, (1 - f) b of the others' averages lands here
        red_hbm = G * f * b + (f * b if shard else b)
        red_nvl = 0.0 if (shard or not multi) else max((world - 1) * f * b, (1 - f) * b)
    else:
        red_hbm = red_nvl = 0.0
    # LAMB, one-pass ideal: read wire grad + p, m, v, write p, m, v; sharded:
    # the fp32 parameters of the owned range go to every other rank
    lamb_hbm = f_l * (24 + b) + ((1 - f) * 4.0 if shard and multi else 0.0)
    lamb_nvl = max((world - 1) * f * 4.0, (1 - f) * 4.0) if (shard and multi) else 0.0
    phases = [(pack_hbm, pack_nvl), (red_hbm, red_nvl), (lamb_hbm, lamb_nvl)]
    return {"f": f, "alg": alg, "impl": impl, "phases": phases,
            "hbm": sum(h for h, _ in phases), "nvl": sum(x for _, x in phases)}


def round_roofline(models, n, peak) -> float:
    """Seconds: HBM and NVLink phases serialized, each on its
    critical-path rank: max_r HBM_r / peak + max_r NVL_r / NVLink."""
    return (max(m["hbm"] for m in models) * n / (peak * 1e9)
            + max(m["nvl"] for m in models) * n / (NVLINK_GBS * 1e9))


def overlap_roofline(models, n, peak) -> float:
    """Seconds, a tighter bound: within each barrier-separated phase (pack +
    scatter, reduce, LAMB [+ parameter push]) HBM and NVLink traffic overlap,
    so the phase costs the slowest rank's max(HBM time, NVLink time)."""
    t = 0.0
    for k in range(3):
        t += max(max(m["phases"][k][0] * n / (peak * 1e9), m["phases"][k][1] * n / (NVLINK_GBS * 1e9))
                 for m in models)
    return t


def choose_shard_lamb(offsets, L: int, world: int, n: int, b: float, wire: str,
                      peak: float = HBM_GBS) -> bool:
    """True when sharded LAMB (owners step, fp32 parameters pushed) has the
    lower round bound than replicated LAMB (averaged gradient pushed, every
    rank steps everything) for this plan, the sharded bound weighted by
    SHARD_PENALTY. Uniform splits favour sharding; a dominant owner
    (het8c's 7/10, het4b's 19/22) pushes 4 B/element instead of b and
    favours replication."""
    if world < 2:
        return False
    t = {}
    for shard in (True, False):
        ms = [rank_model(r, offsets, L, world, n, b, wire, shard, False) for r in range(world)]
        t[shard] = overlap_roofline(ms, n, peak)
    return t[True] * SHARD_PENALTY < t[False]
