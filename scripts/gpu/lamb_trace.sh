mkdir -p gpurun_out
export SP_SKIP_BUILD=1
timeout 300 python scripts/micro/lamb_trace.py build/variants/trace/libsp_round.so albert-large fp16 > gpurun_out/trace_fp16.txt 2>&1
timeout 300 python scripts/micro/lamb_trace.py build/variants/trace/libsp_round.so albert-large q8 > gpurun_out/trace_q8.txt 2>&1
