export SP_SKIP_BUILD=1
N=$(nvidia-smi -L | wc -l)
SP_ROUND_LIB=scripts/variants/libsp_round_occ6.so SP_ROUND_CELL=32768 timeout 600 python -m pytest tests/test_round_gpu.py tests/test_multigpu.py -x -q 2>&1 | tail -2
B="python bench.py --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 5"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 5"
for lib in paper_2106_10207_b200/lib/libsp_round.so scripts/variants/libsp_round_occ6.so; do
for cell in 32768; do for lag in 200 600 1200 100000000; do
  echo "$lib cell=$cell lag=$lag N=1: $(SP_ROUND_LAG=$lag SP_ROUND_LIB=$lib SP_ROUND_CELL=$cell timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'])")"
  echo "$lib cell=$cell lag=$lag N=$N: $(SP_ROUND_LAG=$lag SP_ROUND_LIB=$lib SP_ROUND_CELL=$cell timeout 300 $T 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'])")"
done; done; done
