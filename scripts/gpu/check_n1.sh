mkdir -p gpurun_out
export SP_SKIP_BUILD=1
nvidia-smi -L > gpurun_out/g1_smi.txt 2>&1
timeout 1200 python -m pytest tests/test_round_gpu.py -q --timeout 300 > gpurun_out/g1_test.log 2>&1
echo "pytest rc=$?" >> gpurun_out/g1_test.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
echo "bench rc=$?" >> gpurun_out/g1_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/g1_smoke.log
