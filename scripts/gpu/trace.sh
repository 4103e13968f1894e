# the traced k_lamb timeline (build/variants/trace, SP_LAMB_TRACE)
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
timeout 300 python scripts/micro/lamb_trace.py build/variants/trace/libsp_round.so albert-large fp16 > gpurun_out/it_trace_fp16.txt 2>&1
