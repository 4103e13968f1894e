# ncu --set full (source counters) of one k_lamb launch, N=1 ALBERT-large fp16
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-virtual-peers > gpurun_out/nl_bench.json 2> gpurun_out/nl_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lamb --launch-skip 5 -c 1 -o gpurun_out/ncu_lamb_r2b python bench.py --steps 3 --warmup 3 --phased-steps 1 --no-cpu-baseline --no-virtual-peers > gpurun_out/ncu_lamb_r2b.log 2>&1
[ -x scripts/micro/stream_bw ] && timeout 120 scripts/micro/stream_bw > gpurun_out/nl_stream_bw.txt 2>&1
