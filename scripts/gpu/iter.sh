# one development iteration on the B200: GPU parity tests, the traced LAMB
# timeline, the k_lamb configuration variants
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
timeout 400 python -m pytest tests/test_round_gpu.py tests/test_pybind_round.py -q --timeout 60 -x > gpurun_out/it_test.log 2>&1
echo "pytest rc=$?" >> gpurun_out/it_test.log
timeout 300 python scripts/micro/lamb_trace.py build/variants/trace/libsp_round.so albert-large fp16 > gpurun_out/it_trace_fp16.txt 2>&1
bash scripts/gpu/variants.sh
for i in 1 2; do timeout 300 python scripts/micro/debug_p.py fp16 8 11; done > gpurun_out/dbg_p.txt 2>&1
