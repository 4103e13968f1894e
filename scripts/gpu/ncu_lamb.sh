# ncu --set full (source counters) of one k_lamb launch, N=1 ALBERT-large fp16
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lamb --launch-skip 5 -c 1 -o gpurun_out/ncu_lamb_${1:-x} python bench.py --steps 3 --warmup 3 --phased-steps 1 --no-cpu-baseline --no-virtual-peers > gpurun_out/ncu_lamb_${1:-x}.log 2>&1
