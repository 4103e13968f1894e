# final single-GPU validation: every GPU test, smoke, headline bench, reference arm
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
cat gpurun_out/f_pytest.log gpurun_out/f_smoke.log gpurun_out/f_bench.json gpurun_out/f_ref.json
