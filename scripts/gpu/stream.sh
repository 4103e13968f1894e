# one ncu-free run of the pass-1 bandwidth microbenchmarks
mkdir -p gpurun_out
timeout 300 scripts/micro/stream_bw > gpurun_out/stream_bw.txt 2>&1
