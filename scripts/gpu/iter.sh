# one development iteration on the B200: GPU parity tests, N=1 bench
# (fp16 / q8 / fp32), the traced LAMB timeline, the streaming micro-benchmark
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
[ -x scripts/micro/stream_bw ] && timeout 300 scripts/micro/stream_bw > gpurun_out/it_stream_bw.txt 2>&1
for w in albert-large-fp16 albert-large-q8 albert-large-fp32; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-virtual-peers --workload $w > gpurun_out/it_$w.json 2> gpurun_out/it_$w.err
done
timeout 300 python scripts/micro/lamb_trace.py build/variants/trace/libsp_round.so albert-large fp16 > gpurun_out/it_trace_fp16.txt 2>&1
timeout 1200 python -m pytest tests/test_round_gpu.py tests/test_pybind_round.py -q --timeout 300 -x > gpurun_out/it_test.log 2>&1
echo "pytest rc=$?" >> gpurun_out/it_test.log
