#!/usr/bin/env python
"""BASELINE config 5: scaling sweep of the averaging round over vector size
x wire format at one GPU count, one bench.py line per point.

    python scripts/sweep.py --gpus 1 --out gpurun_out/sweep_n1.jsonl
    python scripts/sweep.py --gpus 4 --out gpurun_out/sweep_n4.jsonl

Each point is `bench.py --workload sweep --params N --wire W` (4 Mi-element
LAMB tensors, homogeneous fleet of N GPUs planned by the LP), launched under
torchrun for N > 1 exactly as the driver launches the headline bench. The
CPU baseline is skipped (the headline bench reports it); everything else in
the line (roofline, e2e, clocks) is the bench's own.
"""
import argparse
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIZES = [1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20, 1 << 30]


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--out", required=True)
    ap.add_argument("--sizes", default=",".join(str(x) for x in SIZES))
    ap.add_argument("--wires", default="fp32,fp16,q8")
    ap.add_argument("--timeout", type=int, default=300, help="per point, seconds")
    args = ap.parse_args()
    bench = os.path.join(ROOT, "bench.py")
    with open(args.out, "a") as out:
        for n in (int(x) for x in args.sizes.split(",")):
            steps = 50 if n <= (64 << 20) else 10
            for wire in args.wires.split(","):
                tail = [bench, "--gpus", str(args.gpus), "--workload", "sweep", "--params", str(n),
                        "--wire", wire, "--steps", str(steps), "--warmup", "3",
                        "--phased-steps", "5", "--no-cpu-baseline"]
                if args.gpus > 1:
                    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
                           f"--master-port={free_port()}", *tail]
                else:
                    cmd = [sys.executable, *tail]
                try:
                    r = subprocess.run(cmd, capture_output=True, text=True, timeout=args.timeout)
                    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
                    if r.returncode != 0 or not lines:
                        rec = {"params": n, "wire": wire, "n_gpus": args.gpus, "error": r.stderr[-800:]}
                    else:
                        rec = json.loads(lines[-1])
                except subprocess.TimeoutExpired:
                    rec = {"params": n, "wire": wire, "n_gpus": args.gpus, "error": "timeout"}
                out.write(json.dumps(rec) + "\n")
                out.flush()
                short = rec.get("round_us"), rec.get("value"), (rec.get("round_roofline") or {}).get("frac")
                print(f"N={args.gpus} params={n} {wire}: round_us, GB/s, roofline frac = {short}",
                      rec.get("error", ""), flush=True)


if __name__ == "__main__":
    main()
