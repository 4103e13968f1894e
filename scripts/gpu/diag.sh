# micro + k_lamb variants (build/variants/*) on one box
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
timeout 300 scripts/micro/stream_bw > gpurun_out/stream_bw.txt 2>&1
bash scripts/gpu/variants.sh
