# the albert-large G=8 fp16 parity case (step by step, mismatches grouped by tensor)
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
for i in 1 2 3; do timeout 300 python scripts/micro/debug_p.py fp16 8 11; done > gpurun_out/dbg_p.txt 2>&1
timeout 300 python scripts/micro/debug_p.py q8 8 11 >> gpurun_out/dbg_p.txt 2>&1
timeout 300 python scripts/micro/debug_p.py fp32 8 11 >> gpurun_out/dbg_p.txt 2>&1
