# q8 parity tests and N=1 q8/fp16 bench lines
mkdir -p gpurun_out/q8
export SP_SKIP_BUILD=1
timeout 600 python -m pytest tests/test_round_gpu.py -q --timeout 120 -k "q8" > gpurun_out/q8/test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q8/test.log
for w in albert-large-q8 resnet50-q8 albert-large-fp16; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-virtual-peers --workload $w > gpurun_out/q8/n1_$w.json 2> gpurun_out/q8/n1_$w.err
done
timeout 300 python scripts/micro/debug_p.py q8 8 11 > gpurun_out/q8/dbg.txt 2>&1
