set -x
export SP_SKIP_BUILD=1
SP_LAMB_L2HINTS=1 timeout 900 python -m pytest tests/test_round_gpu.py -x -q 2>&1 | tail -3
B="python bench.py --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 10"
for h in 0 1; do
for lag in 150 300 600 1200 100000; do
  echo "hints=$h lag=$lag"; SP_LAMB_L2HINTS=$h SP_LAMB_LAG=$lag timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'], d['kernel_ms']['moments_ms'])"
done; done
