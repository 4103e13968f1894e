export SP_SKIP_BUILD=1
B="python bench.py --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 5"
run() { echo "$* : $(env "$@" timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'], round(d['kernel_ms']['moments_ms']*1000,1))")"; }
SP_ROUND_LIB=scripts/variants/libsp_round_t512.so timeout 300 python -m pytest tests/test_round_gpu.py -q -x 2>&1 | tail -1
for lib in paper_2106_10207_b200/lib/libsp_round.so scripts/variants/libsp_round_t512.so; do
for grid in 296 592 100000; do for ch in 4096 8192; do for lag in 300 800 1000000000; do
run SP_ROUND_LIB=$lib SP_LAMB_GRID=$grid SP_LAMB_CHUNK=$ch SP_LAMB_LAG=$lag
done; done; done; done
