# every N=1 bench workload (one B200)
mkdir -p gpurun_out/wl
export SP_SKIP_BUILD=1
for w in albert-large-fp16 albert-large-fp32 albert-large-q8 albert-base-fp32 resnet50-q8 het8c-fp16 het4b-fp32; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --workload $w > gpurun_out/wl/n1_$w.json 2> gpurun_out/wl/n1_$w.err
done
