# hybrid sharded LAMB: parity (sharded multi-GPU tests, forced split) and a sweep of the split
export SP_SKIP_BUILD=1
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
SP_SHARD_FRACTION=0.5 timeout 600 python -m pytest tests/test_multigpu.py -x -q -k shard 2>&1 | tail -2
timeout 600 python -m pytest tests/test_multigpu.py -x -q -k shard 2>&1 | tail -2
for wl in albert-large-fp16 albert-large-fp32 albert-large-q8; do
for fr in auto 1.0 0.7 0.5 0.3; do
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 10 --shard-lamb --workload $wl"
  if [ $fr = auto ]; then out=$(timeout 300 $T 2>/dev/null | grep '^{'); else out=$(SP_SHARD_FRACTION=$fr timeout 300 $T 2>/dev/null | grep '^{'); fi
  echo "N=$N $wl shard=$fr: $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'], d['config'].get('shard_cut'), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})")"
done
done
