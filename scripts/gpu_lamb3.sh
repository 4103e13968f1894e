export SP_SKIP_BUILD=1
B="python bench.py --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 10"
for lib in paper_2106_10207_b200/lib/libsp_round.so scripts/variants/libsp_round_lamb6.so scripts/variants/libsp_round_lamb8.so; do
  echo "$lib: $(SP_ROUND_LIB=$lib timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'], round(d['kernel_ms']['moments_ms']*1000,1))")"
  echo "$lib g8: $(SP_ROUND_LIB=$lib timeout 300 $B --peers-per-gpu 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'], round(d['kernel_ms']['moments_ms']*1000,1), round(d['kernel_ms']['reduce_ms']*1000,1), round(d['kernel_ms']['pack_ms']*1000,1))")"
done
SP_ROUND_LIB=scripts/variants/libsp_round_lamb8.so timeout 300 python -m pytest tests/test_round_gpu.py -q -x 2>&1 | tail -1
