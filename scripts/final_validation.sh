set -x
mkdir -p gpurun_out/final
nvidia-smi -L > gpurun_out/final/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/final/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/final/smoke.log
timeout 600 python bench.py > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err; echo "bench exit $?" >> gpurun_out/final/bench_n1.err
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
tail -3 gpurun_out/final/pytest_gpu.log; cat gpurun_out/final/bench_n1.json gpurun_out/final/bench_ref.json | cut -c1-600
