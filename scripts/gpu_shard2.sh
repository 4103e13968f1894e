# sharded LAMB push-kernel sweep at N GPUs (fp16), plus parity of the sharded tests
export SP_SKIP_BUILD=1
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_multigpu.py -x -q -k shard 2>&1 | tail -2
for ch in 8192 4096 16384; do
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 10 --shard-lamb"
  out=$(SP_LAMB_CHUNK=$ch timeout 300 $T 2>/dev/null | grep '^{')
  echo "N=$N shard chunk=$ch: $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'], d['kernel_ms'])")"
done
