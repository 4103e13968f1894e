# Sharded vs replicated LAMB at N GPUs (N = visible GPUs), per wire format.
export SP_SKIP_BUILD=1
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for wl in albert-large-fp16 albert-large-fp32 albert-large-q8; do
  for mode in "" "--shard-lamb"; do
    T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 10 --workload $wl $mode"
    out=$(timeout 300 $T 2>gpurun_out/shard_err.log | grep '^{')
    echo "$out" > "gpurun_out/bench_n${N}_${wl}${mode}.json"
    echo "N=$N $wl ${mode:-replicated}: $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'], d['kernel_ms'], d['round_roofline'])")"
  done
done
