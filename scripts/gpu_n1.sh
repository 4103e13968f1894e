export SP_SKIP_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for w in albert-large-fp16 albert-large-fp32 albert-large-q8; do
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 10 --workload $w > gpurun_out/b_$w.json 2>/dev/null
  echo "$w $(python -c "import json; d=json.load(open('gpurun_out/b_$w.json')); print(d['round_us'], d['gpu_launches'], d['roofline']['frac'], d['round_roofline'], {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})")"
done
SP_NO_FUSED_PACK=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 10 > gpurun_out/b_nofuse.json 2>/dev/null
echo "fp16 no fused pack $(python -c "import json; d=json.load(open('gpurun_out/b_nofuse.json')); print(d['round_us'])")"
