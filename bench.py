#!/usr/bin/env python
"""Benchmark of the DeDLOC averaging round (grad avg + LAMB step) on B200.

One step = one butterfly averaging round over a flattened gradient vector
(pack -> reduce-scatter / weighted average / all-gather over NVLink -> LAMB)
through libsp_round.so. Default workload: ALBERT-large-sized vector
(17,847,474 params, 32-tensor LAMB table), fp16 wire, one peer per GPU
(G = N, weak scaling), LP-balanced fractions, synthetic gradients.

    python bench.py --gpus 1 --steps 50 --warmup 5
    torchrun --nproc-per-node 8 ... bench.py --gpus 8 --steps 50 --warmup 5
    python bench.py --impl reference ...   # reference run_plan + oracle LAMB on host cores

Prints ONE JSON line on rank 0 (stdout); diagnostics go to stderr.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "averaging round time + GB/s (grad avg + LAMB step), ALBERT-large, 1/2/4/8 B200"
HP = dict(lr=1.76e-3, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.01, bias_correction=1)
SIGMA = 1e-3 * 3 ** 0.5
L2_BYTES = 126e6

WORKLOADS = {
    # name: (tensor table, wire, q8 block, fleet). fleet None: G homogeneous
    # peers; otherwise a named collaboration (paper_2106_10207_b200/fleets.py)
    # whose peer count fixes G. Either way the LP (solve_strategy) plans the
    # round: fractions -> part offsets, sample counts -> weights.
    "albert-large-fp16": ("albert-large", "fp16", 4096, None),
    "albert-large-fp32": ("albert-large", "fp32", 4096, None),
    "albert-large-q8": ("albert-large", "q8", 4096, None),
    "resnet50-q8": ("resnet50", "q8", 4096, None),
    "albert-base-fp32": ("albert-base", "fp32", 4096, None),
    # BASELINE config 1 (reference CPU scenario): ALBERT-base, fp32, 4 heterogeneous peers
    "het4b-fp32": ("albert-base", "fp32", 4096, "het4b"),
    # BASELINE config 4: 8 peers incl. a client, fractions 1/20 x6, 0, 7/10
    "het8c-fp16": ("albert-large", "fp16", 4096, "het8c"),
    # BASELINE config 5: --params N, --wire {fp32,fp16,q8}; 4 Mi-element tensors
    "sweep": ("uniform4m", None, 4096, None),
}
TARGET_BATCH = 4096.0  # PAPER.md:842; the LP's sample counts are scaled to it


def log(*a):
    print(*a, file=sys.stderr, flush=True)


_STDOUT_FD = None


def quiet_stdout() -> None:
    """Route fd 1 to stderr for the whole run (NCCL and library banners
    print there) and keep the real stdout for the one JSON line."""
    global _STDOUT_FD
    if _STDOUT_FD is None:
        sys.stdout.flush()
        _STDOUT_FD = os.dup(1)
        os.dup2(2, 1)


def emit(obj) -> None:
    line = (json.dumps(obj) + "\n").encode()
    if _STDOUT_FD is None:
        sys.stdout.write(line.decode())
        sys.stdout.flush()
    else:
        os.write(_STDOUT_FD, line)


def tensor_table(name: str, params: int = 0) -> list[int]:
    if name == "uniform4m":  # sweep: 4,194,304-element tensors, remainder last
        if params < 1:
            raise SystemExit("--workload sweep needs --params N")
        t = 4 * 1024 * 1024
        return [t] * (params // t) + ([params % t] if params % t else [])
    with open(os.path.join(ROOT, "tests", "golden", "tensor_tables.json")) as f:
        return json.load(f)[name]


def wire_bytes(wire: str, block: int) -> float:
    return {"fp32": 4.0, "fp16": 2.0, "q8": 1.0 + 4.0 / block}[wire]


def ncu_traffic(kernel_substr: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of the kernel in the
    newest committed `ncu --set full` capture (profiles/*/ncu_full_*.csv),
    bytes per launch, or None when no capture of that kernel is committed."""
    import csv
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_full_*.csv")), reverse=True):
        try:
            rows = list(csv.reader(open(path)))
            h = rows[0]
            ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
            unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            ur, uw = unit.get(rows[1][ri], 1.0), unit.get(rows[1][wi], 1.0)
            for r in rows[2:]:
                if kernel_substr in r[ki]:
                    return float(r[ri]) * ur + float(r[wi]) * uw
        except Exception:
            continue
    return None


def peak_hbm() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms (recipe's line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows: list[list[str]] = []
        self.proc = None
        self.marks: list[tuple[float, float]] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception as e:  # nvidia-smi missing: report empty clocks
            log("clock sampler unavailable:", e)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([time.time()] + [x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        rows = self.rows
        if self.marks:
            t0, t1 = self.marks[0]
            inside = [r for r in rows if t0 - 0.25 <= r[0] <= t1 + 0.25]
            rows = inside or rows
        sm = [float(r[2]) for r in rows if len(r) > 3 and r[2].replace(".", "").isdigit()]
        smax = [float(r[3]) for r in rows if len(r) > 3 and r[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for k, nm in enumerate(names):
                if len(r) > 6 + k and r[6 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ---------------------------------------------------------- CPU reference
def make_cpu_round(tsizes, wire, block, G, weights):
    """The path on the host: every peer's gradient packed to the wire format
    (oracle), the weighted mean of the wire buffers by the REFERENCE's own
    groups::run_plan (oracle/_ref: /root/reference/proj/src/groups.cpp
    compiled unmodified; fp64, peer order), the mean rounded to the wire
    format (oracle) and the LAMB step (oracle; the reference has no LAMB,
    SPEC.md:519). Returns one(step, threads) -> per-phase seconds."""
    import numpy as np

    from oracle import oracle as O
    from oracle import ref as R

    n = sum(tsizes)
    grads = [None if weights[g] == 0 else O.fill_synthetic(n, 1, g, SIGMA) for g in range(G)]
    p = O.fill_synthetic(n, 2, 0, 0.02, 0)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    mean = np.empty(n, np.float64)

    def one(step: int, threads: int) -> dict:
        O.set_threads(threads)
        t0 = time.perf_counter()
        packed = [None if x is None else O.pack(wire, x, block) for x in grads]
        t1 = time.perf_counter()
        R.weighted_mean_wire(wire, packed, weights, block, threads=threads, out=mean)
        t2 = time.perf_counter()
        avg, avg_s = O.wire_from_f64(wire, mean, block)
        t3 = time.perf_counter()
        O.lamb(wire, avg, avg_s, p, m, v, tsizes, HP, step, block)
        t4 = time.perf_counter()
        return {"pack_s": t1 - t0, "average_s": t2 - t1, "to_wire_s": t3 - t2, "lamb_s": t4 - t3,
                "round_s": t4 - t0}

    return one


def host_threads() -> int:
    return len(os.sched_getaffinity(0))  # every host core (torchrun sets OMP_NUM_THREADS=1)


def cpu_baseline(tsizes, wire, block, G, weights, grad_bytes, budget_s: float = 30.0) -> dict:
    """the CPU path in two modes, 1 thread (the reference is
    single-threaded, proj/CMakeLists.txt:12) and every host core; median of
    10 rounds after 2 warm-ups (fewer rounds when 12 would exceed the time
    budget: the sample stays bounded)."""
    one = make_cpu_round(tsizes, wire, block, G, weights)
    modes = {}
    step = 0
    for label, th in (("1_thread", 1), ("all_cores", host_threads())):
        step += 1
        t_first = one(step, th)["round_s"]  # warm-up 1
        step += 1
        one(step, th)  # warm-up 2
        reps = int(max(3, min(10, budget_s / 2 / max(t_first, 1e-6))))
        runs = []
        for _ in range(reps):
            step += 1
            runs.append(one(step, th))
        med = {k: statistics.median(r[k] for r in runs) for k in runs[0]}
        modes[label] = {"threads": th, "rounds": reps,
                        "round_ms": round(med["round_s"] * 1e3, 3),
                        "value": round(grad_bytes / med["round_s"] / 1e9, 4),
                        "phase_ms": {k.replace("_s", "_ms"): round(x * 1e3, 3) for k, x in med.items()
                                     if k != "round_s"}}
    best = modes["all_cores"]
    return {"value": best["value"], "unit": "GB/s", "cores": best["threads"], "kind": "reference",
            "round_ms": best["round_ms"], "cpu_model": cpu_model(), "modes": modes,
            "sample": f"full {len(tsizes)}-tensor vector ({sum(tsizes)} params), G={G}, {wire} wire: "
                      "oracle pack -> reference groups::run_plan weighted mean (oracle/_ref, "
                      "column blocks over threads) -> wire -> oracle LAMB; median of "
                      f"{modes['1_thread']['rounds']} (1 thread) / {best['rounds']} (all cores) "
                      "rounds after 2 warm-ups"}


def lp_solve_times() -> dict:
    """Host LP (strategy solve) time, median of 5, for the fleets the budget is
    quoted on (< 50 ms at n = 16: PAPER.md:140)."""
    from paper_2106_10207_b200 import _swarmplan
    from paper_2106_10207_b200.fleets import homogeneous, spec_json

    out = {}
    for name, sj in (("n4_homogeneous", json.dumps(homogeneous(4, 1.0, 1000.0, 4.0, 17847474))),
                     ("n8_homogeneous8", spec_json("homogeneous8")),
                     ("n8_het8c", spec_json("het8c")),
                     ("n16_static16", spec_json("static16")),
                     ("n16_table1_b", spec_json("table1_b"))):
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            _swarmplan.solve_strategy(sj)
            ts.append(time.perf_counter() - t0)
        out[name] = round(statistics.median(ts) * 1e3, 2)
    return out


from paper_2106_10207_b200.roofline import (NVLINK_GBS, overlap_roofline, rank_model,  # noqa: E402,F401
                                            round_roofline)


def dominant_kernel(ph: dict, model: dict, world: int, L: int, n: int, b: float, shard: bool,
                    peak: float) -> dict:
    """Roofline of the longest kernel of one rank's phased round: §8(d)
    algorithmic bytes of one launch / its event-timed duration."""
    f_r, alg = model["f"], model["alg"]
    dom = max(("pack_ms", "reduce_ms", "lamb_ms"), key=lambda k: ph[k])
    achieved = alg[dom] / (ph[dom] * 1e-3) / 1e9
    bound, pk = "hbm", peak
    if shard and dom == "lamb_ms" and world > 1:  # parameter push: (world-1) f 4 B out
        bound, pk = "nvlink", NVLINK_GBS
        achieved = (world - 1) * f_r * 4.0 * n / (ph[dom] * 1e-3) / 1e9
    elif dom in ("reduce_ms", "pack_ms") and world > 1:
        bound, pk = "nvlink", NVLINK_GBS
        # per direction: pack scatters L (1-f) b n, reduce pushes (world-1) f b n
        nvl = (L * (1 - f_r) * b * n) if dom == "pack_ms" else ((world - 1) * f_r * b * n)
        achieved = nvl / (ph[dom] * 1e-3) / 1e9
    return {"kernel": dom, "bound": bound, "achieved": achieved, "peak": pk}


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="albert-large-fp16")
    ap.add_argument("--peers-per-gpu", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-virtual-peers", action="store_true",
                    help="skip the N=1 8-virtual-peer pass (pack + reduce timed)")
    ap.add_argument("--phased-steps", type=int, default=20)
    ap.add_argument("--lamb", choices=["auto", "replicated", "sharded"], default="auto",
                    help="replicated: every GPU steps the all-gathered average; sharded: ZeRO-1 "
                         "style, owners step their range and push fp32 parameters; auto: at N > 1 "
                         "the mode with the lower round bound for the LP plan "
                         "(roofline.choose_shard_lamb: sharded for uniform splits, replicated "
                         "when one owner dominates)")
    ap.add_argument("--shard-lamb", action="store_true", help="alias of --lamb sharded")
    ap.add_argument("--params", type=int, default=0, help="--workload sweep: vector length")
    ap.add_argument("--wire", choices=["fp32", "fp16", "q8"], default=None,
                    help="override the workload's wire format (required for sweep)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    quiet_stdout()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.shard_lamb:
        args.lamb = "sharded"
    args.shard_lamb = args.lamb == "sharded"  # auto: decided from the plan below
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"note: WORLD_SIZE={world} but --gpus={args.gpus}; using WORLD_SIZE")

    table, wire, block, fleet = WORKLOADS[args.workload]
    wire = args.wire or wire
    if wire is None:
        raise SystemExit(f"--workload {args.workload} needs --wire")
    tsizes = tensor_table(table, args.params)
    n = sum(tsizes)
    from paper_2106_10207_b200 import fleets
    from paper_2106_10207_b200.dist import plan_round

    if fleet:
        spec_j = fleets.spec_json(fleet)
        n_peers = len(json.loads(spec_j)["peers"])
        if n_peers % world:
            raise SystemExit(f"fleet {fleet} has {n_peers} peers; WORLD_SIZE={world} must divide it")
        L = n_peers // world
    else:
        L = args.peers_per_gpu
        spec_j = json.dumps(fleets.homogeneous(L * world, 1.0, 1000.0, TARGET_BATCH, n))
    G = L * world
    # host LP plan (every rank solves the same deterministic program;
    # AveragingRound.set_assignment checks they agree)
    align = block if wire == "q8" else 8  # sp_round_align: no q8 block straddles owners
    plan = plan_round(spec_j, n, align)
    offsets = [int(x) for x in plan["offsets"]]
    wsum = sum(plan["weights"])
    weights = [w * TARGET_BATCH / wsum for w in plan["weights"]]  # sample counts, sum = batch
    b = wire_bytes(wire, block)
    if args.lamb == "auto":
        from paper_2106_10207_b200.roofline import choose_shard_lamb

        args.shard_lamb = choose_shard_lamb(offsets, L, world, n, b, wire)

    if args.impl == "reference":
        return run_reference(args, rank, world, tsizes, wire, block, G, weights)

    if os.environ.get("NCCL_DEBUG", "VERSION").upper() in ("VERSION", ""):
        os.environ["NCCL_DEBUG"] = "WARN"  # keep stdout to the one JSON line
    import torch

    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2106_10207_b200 import AveragingRound, fill_synthetic

    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(dev)

    def make_round(peers, shard):
        return AveragingRound(n, tsizes, wire=wire, q8_block=block, peers_per_rank=peers, rank=rank,
                              world=world, device=local_rank, lr=HP["lr"],
                              betas=(HP["beta1"], HP["beta2"]), eps=HP["eps"],
                              weight_decay=HP["weight_decay"], shard_lamb=shard)

    rnd = make_round(L, args.shard_lamb)
    if rnd.align != align:
        raise SystemExit(f"align mismatch: library {rnd.align}, planned {align}")
    rnd.set_assignment(offsets, weights)
    grads = []
    for l in range(L):
        g = torch.empty(n, dtype=torch.float32, device=dev)
        fill_synthetic(g, 1, rank * L + l, SIGMA)
        grads.append(g)
    p = rnd.param_buffer() if args.shard_lamb else torch.empty(n, dtype=torch.float32, device=dev)
    fill_synthetic(p, 2, 0, 0.02, 0)
    m = torch.zeros(n, dtype=torch.float32, device=dev)
    v = torch.zeros(n, dtype=torch.float32, device=dev)
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    step = 0

    def one():
        nonlocal step
        step += 1
        rnd.run(grads, p, m, v, step, stream)

    clocks = ClockSampler(local_rank)
    clocks.start()
    # warm-up: W steps, then keep stepping (untimed) for >= 1 s so clocks ramp
    # and the sampler has samples under load
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            one()
        torch.cuda.synchronize(dev)
        t_end = time.time() + 1.0
        while time.time() < t_end:
            for _ in range(20):
                one()
            stream.synchronize()
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        wall0 = time.time()
        e0.record(stream)
        for _ in range(args.steps):
            one()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        wall1 = time.time()
        barrier()
        # keep the load on for the sampler if the timed region was short
        t_end = time.time() + max(0.0, 0.6 - (wall1 - wall0))
        while time.time() < t_end:
            for _ in range(20):
                one()
            stream.synchronize()
        torch.cuda.synchronize(dev)
    clocks.marks.append((wall0, max(wall1, wall0 + 0.6)))
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    grad_bytes = 4.0 * n * G  # fp32 gradient bytes of all peers averaged per round
    value = grad_bytes / (ms_step * 1e-3) / 1e9

    # per-kernel device times (non-graph pass with events between kernels)
    def phased(r, gs, pp, mm, vv, k):
        nonlocal step
        out = []
        with torch.cuda.stream(stream):
            for _ in range(k):
                step += 1
                out.append(r.run_phased(gs, pp, mm, vv, step, stream))
        return {key: statistics.median(x[key] for x in out) for key in out[0]}

    ph = phased(rnd, grads, p, m, v, args.phased_steps)

    # e2e through the public API with host buffers: H2D of this rank's
    # accumulated gradients from pinned memory into double-buffered device
    # staging (step k's copy overlaps round k-1), the round, and the D2H of
    # the step's result, the updated parameters (p_out). PCIe is full
    # duplex, so the parameter read-back overlaps the next upload.
    host_g = [gg.cpu().pin_memory() for gg in grads]
    p_host = torch.empty(n, dtype=torch.float32).pin_memory()
    e2e_steps = max(3, min(args.steps, 20))

    def one_host():
        nonlocal step
        step += 1
        rnd.run_host(host_g, p, m, v, step, stream, p_out=p_host)

    with torch.cuda.stream(stream):
        for _ in range(3):  # captures the graphs of both staging buffers
            one_host()
        barrier()
        torch.cuda.synchronize(dev)
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(e2e_steps):
            one_host()
        f1.record(stream)
        torch.cuda.synchronize(dev)
    e2e_ms = f0.elapsed_time(f1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_step = e2e_ms / e2e_steps
    e2e_value = grad_bytes / (e2e_step * 1e-3) / 1e9

    all_ph = [ph]
    if world > 1:
        all_ph = [None] * world
        torch.distributed.all_gather_object(all_ph, ph)
    nchunks = rnd.lamb_chunks()[0]
    rnd.close()
    del host_g, p_host

    # N=1 only: the same vector split over 8 virtual peers on this GPU, so
    # that the pack and the weighted reduce (which a one-peer round skips)
    # are timed in the driver's own bench run too
    virt = None
    if world == 1 and L == 1 and not args.no_virtual_peers:
        try:
            virt = virtual_peer_pass(make_round, n, wire, b, dev, stream, args, fill_synthetic)
        except Exception as e:  # a diagnostic; never fails the bench line
            log("virtual-peer pass failed:", e)

    if rank == 0:
        peak, peak_kind = peak_hbm()
        shard = args.shard_lamb
        # one GPU, one peer, fp32/fp16: the pack runs inside LAMB pass 1
        fused_pack = world == 1 and L == 1 and wire != "q8"
        models = [rank_model(r, offsets, L, world, n, b, wire, shard, fused_pack)
                  for r in range(world)]
        # critical rank: the one with the longest modeled round (non-uniform
        # LP splits put the big owner on the critical path);
        # every rank's phased times include waiting for it at the barriers
        rc = max(range(world), key=lambda r: (round_roofline([models[r]], n, peak), -r))
        phc, mc = all_ph[rc], models[rc]
        dk = dominant_kernel(phc, mc, world, L, n, b, shard, peak)
        dom = dk["kernel"]
        widx = {"fp32": 0, "fp16": 1, "q8": 2}[wire]
        fused = world == 1 and L == 1 and wire != "q8"  # the pack runs inside k_lamb<W, true>
        kname = {"pack_ms": f"k_pack_{wire}", "reduce_ms": f"k_reduce_{wire}",
                 "lamb_ms": f"k_lamb<{widx}, {int(fused)}>"}[dom]
        traffic = (ncu_traffic(kname) if table == "albert-large" and world == 1 and L == 1 else None)
        # whole-round roofline (per phase on the slowest rank)
        hbm_round = max(x["hbm"] for x in models)
        nvl_round = max(x["nvl"] for x in models)
        t_roof = round_roofline(models, n, peak)
        t_ovl = overlap_roofline(models, n, peak)
        lp_times = None
        try:
            lp_times = lp_solve_times()
        except Exception as e:
            log("lp timing failed:", e)
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                cpu = cpu_baseline(tsizes, wire, block, G, weights, grad_bytes)
            except Exception as e:
                log("cpu baseline failed:", e)
        fr = [round(x, 6) for x in plan["fractions"]]
        alg_b = mc["alg"].get(dom)
        out = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 5),
            "round_us": round(ms_step * 1e3, 2),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": {"fp32": "f32", "fp16": "f16 wire / f32 accum", "q8": "u8 wire / f32 accum"}[wire],
            "data": "synthetic (counter-hash gradients, sigma=1e-3, 1/997 outliers x100)",
            "config": {"workload": f"{args.workload}: DeDLOC butterfly round + LAMB",
                       "params": n, "tensors": len(tsizes), "peers": G, "peers_per_gpu": L,
                       "wire": wire, "q8_block": block if wire == "q8" else None,
                       "lamb": "sharded (ZeRO-1: owners step, fp32 params pushed)" if args.shard_lamb
                               else "replicated (averaged gradient all-gathered)",
                       "lamb_chunks": nchunks,
                       "fleet": fleet or f"homogeneous{G}",
                       "fractions": fr if G <= 16 else f"{min(fr)}..{max(fr)}",
                       "plan": "solve_strategy (host LP) -> part_offsets; weights = LP sample "
                               f"counts scaled to batch {TARGET_BATCH:g}",
                       "l2": f"no flush: per-step working set {(n * (12 + 4 * L + 2 * b)) / 1e9:.2f} GB > 126 MB L2",
                       "parallelism": f"dp{world} (one process per GPU, {L} peer(s) each, CUDA IPC over NVLink)"},
            # pack (fused into LAMB on one GPU with one peer) + reduce (G > 1)
            # + k_lamb + barriers (N > 1: after the scatter, and after the
            # push of the averages (replicated) or of the parameters (sharded))
            "gpu_launches": args.steps * ((0 if fused_pack else 1) + (1 if G > 1 else 0) + 1
                                          + (2 if world > 1 else 0)),
            "kernel_ms": {k: round(v_, 5) for k, v_ in ph.items()},
            "kernel_ms_critical_rank": {k: round(v_, 5) for k, v_ in phc.items()} if rc else None,
            "roofline": {"bound": dk["bound"], "kernel": kname, "rank": rc,
                         "achieved": round(dk["achieved"], 1), "peak": dk["peak"], "unit": "GB/s",
                         "frac": round(dk["achieved"] / dk["peak"], 4),
                         "traffic": traffic,
                         "traffic_over_alg": round(traffic / alg_b, 4) if traffic and alg_b else None,
                         "algorithmic_bytes": alg_b,
                         "algorithmic_B_per_param": round(alg_b / n, 3) if alg_b else None,
                         "kernel_bytes": mc["impl"].get(dom),
                         "peak_kind": peak_kind if dk["bound"] == "hbm" else
                                      "measured peer copy per direction (B200_PROFILING.md)"},
            # primary: the overlap bound (a lower bound on the round time; the
            # §8d serialized sum is not one: large N=4 rounds beat it)
            "round_roofline": {"t_roof_us": round(t_ovl * 1e6, 2),
                               "frac": round(t_ovl * 1e3 / ms_step, 4),
                               "hbm_B_per_param": round(hbm_round, 3),
                               "nvlink_B_per_param_dir": round(nvl_round, 3),
                               "model": f"sum over barrier-separated phases (pack+scatter, reduce, "
                                        f"LAMB[+param push]) of the slowest rank's max(HBM B/{peak:g}, "
                                        f"NVLink B/{NVLINK_GBS:g} GB/s)",
                               "t_roof_serialized_us": round(t_roof * 1e6, 2),
                               "frac_serialized": round(t_roof * 1e3 / ms_step, 4)},
            "virtual_peers_n1": virt,
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s",
                    "round_us": round(e2e_step * 1e3, 2),
                    "h2d_bytes_per_step": 4 * n * L, "d2h_bytes_per_step": 4 * n,
                    "api": "AveragingRound.run_host(p_out=) -> sp_round_run_host_params (pinned host "
                           "gradients in, updated parameters out; step k's H2D overlaps round k-1 "
                           "and the D2H of step k-1)"},
            "clocks": clk,
            "cpu_baseline": cpu,
            "lp_solve_ms": lp_times,
        }
        emit(out)
    if world > 1:
        torch.distributed.destroy_process_group()


def virtual_peer_pass(make_round, n, wire, b, dev, stream, args, fill_synthetic) -> dict:
    """One GPU hosting all 8 peers of a uniform fleet: times the round and,
    from a phased pass, the pack, reduce and LAMB kernels against §8(d)."""
    import torch

    Gv = 8
    rv = make_round(Gv, False)
    rv.assign([1.0 / Gv] * Gv, [TARGET_BATCH / Gv] * Gv)
    gv = []
    for l in range(Gv):
        t_ = torch.empty(n, dtype=torch.float32, device=dev)
        fill_synthetic(t_, 1, l, SIGMA)
        gv.append(t_)
    pv = torch.empty(n, dtype=torch.float32, device=dev)
    fill_synthetic(pv, 2, 0, 0.02, 0)
    mv, vv = torch.zeros_like(pv), torch.zeros_like(pv)
    step = 0
    with torch.cuda.stream(stream):
        for _ in range(3):
            step += 1
            rv.run(gv, pv, mv, vv, step, stream)
        torch.cuda.synchronize(dev)
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0.record(stream)
        for _ in range(args.steps):
            step += 1
            rv.run(gv, pv, mv, vv, step, stream)
        v1.record(stream)
        torch.cuda.synchronize(dev)
        vms = v0.elapsed_time(v1) / args.steps
        out = []
        for _ in range(args.phased_steps):
            step += 1
            out.append(rv.run_phased(gv, pv, mv, vv, step, stream))
    vph = {key: statistics.median(x[key] for x in out) for key in out[0]}
    model = rank_model(0, rv.offsets, Gv, 1, n, b, wire, False, False)
    peak = peak_hbm()[0]
    kern = {}
    for k in ("pack_ms", "reduce_ms", "lamb_ms"):
        gbs = model["alg"][k] / (vph[k] * 1e-3) / 1e9
        kern[k.replace("_ms", "")] = {"ms": round(vph[k], 5), "algorithmic_bytes": model["alg"][k],
                                      "achieved_gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}
    rv.close()
    return {"peers": Gv, "round_us": round(vms * 1e3, 2),
            "value": round(4.0 * n * Gv / (vms * 1e-3) / 1e9, 3), "unit": "GB/s", "kernels": kern,
            "note": "N=1 with 8 virtual peers (one GPU holds all 8 peers' gradients): §8(d) bytes, "
                    "pack 4+b per peer element, reduce G f b + f b, LAMB 24+b"}


def run_reference(args, rank, world, tsizes, wire, block, G, weights):
    """--impl reference: the path on the host cores with the reference's own
    code where it exists (groups::run_plan from oracle/_ref, column blocks
    spread over every host thread) and the oracle for what the reference
    lacks (wire pack, LAMB). Rank 0 only."""
    if rank != 0:
        return 0
    n = sum(tsizes)
    reps = max(1, args.steps)
    threads = host_threads()
    one = make_cpu_round(tsizes, wire, block, G, weights)
    for w in range(args.warmup):
        one(w + 1, threads)
    runs = [one(args.warmup + r + 1, threads) for r in range(reps)]
    sec = statistics.mean(r["round_s"] for r in runs)
    grad_bytes = 4.0 * n * G
    val = grad_bytes / sec / 1e9
    phase = {k.replace("_s", "_ms"): round(statistics.median(r[k] for r in runs) * 1e3, 3)
             for k in runs[0] if k != "round_s"}
    out = {
        "metric": METRIC, "impl": "reference", "value": round(val, 4), "unit": "GB/s",
        "n_gpus": world, "steps": reps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {"fp32": "f32", "fp16": "f16 wire / f32 accum", "q8": "u8 wire / f32 accum"}[wire],
        "data": "synthetic",
        "config": {"workload": f"{args.workload}: DeDLOC butterfly round + LAMB", "params": n,
                   "tensors": len(tsizes), "peers": G, "peers_per_gpu": G // max(world, 1),
                   "wire": wire},
        "phase_ms": phase,
        "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"full vector, G={G} peers on the host, {reps} rounds: oracle pack -> "
                                   "reference groups::run_plan (oracle/_ref) -> wire -> oracle LAMB"},
        "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(out)
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
