# the bulk-copy staging microbenchmark
mkdir -p gpurun_out
timeout 300 scripts/micro/tma_stream > gpurun_out/tma_stream.txt 2>&1
