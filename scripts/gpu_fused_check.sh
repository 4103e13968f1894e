set -x
export SP_SKIP_BUILD=1
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_round_gpu.py -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -3
B="python bench.py --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 10"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 10"
for mode in 0 1; do
  echo "legacy=$mode N=1"; SP_ROUND_LEGACY=$mode timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'], d['kernel_ms'])"
  echo "legacy=$mode N=$N"; SP_ROUND_LEGACY=$mode timeout 300 $T 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'], d['kernel_ms'])"
done
