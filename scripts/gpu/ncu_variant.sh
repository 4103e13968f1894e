# ncu --set full (source counters) of one k_lamb launch of a variant build
# ($1 = build/variants/<name>), N=1 ALBERT-large fp16
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
V=$1
cp $V/libsp_round.so paper_2106_10207_b200/lib/libsp_round.so
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lamb --launch-skip 5 -c 1 -o gpurun_out/ncu_$(basename $V) python bench.py --steps 3 --warmup 3 --phased-steps 1 --no-cpu-baseline --no-virtual-peers > gpurun_out/ncu_$(basename $V).log 2>&1
