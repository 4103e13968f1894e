# build/variants/*/libsp_round.so (k_lamb compile-time configurations, built
# locally): N=1 bench per variant, then the GPU parity tests of the default
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
LIB=paper_2106_10207_b200/lib/libsp_round.so
cp $LIB /tmp/default.so
for v in build/variants/c*; do
  cp $v/libsp_round.so $LIB
  for w in albert-large-fp16 albert-large-q8; do
    timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-virtual-peers --workload $w > gpurun_out/va_$(basename $v)_$w.json 2> gpurun_out/va_$(basename $v)_$w.err
  done
done
cp /tmp/default.so $LIB
timeout 300 python scripts/micro/lamb_trace.py build/variants/trace/libsp_round.so albert-large fp16 > gpurun_out/va_trace_fp16.txt 2>&1
timeout 1200 python -m pytest tests/test_round_gpu.py -q --timeout 300 -x > gpurun_out/va_test.log 2>&1
echo "pytest rc=$?" >> gpurun_out/va_test.log
