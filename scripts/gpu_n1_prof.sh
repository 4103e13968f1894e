# N=1: GPU tests, headline bench, launch list + one full ncu capture of the top kernel, NVLS probe
set -x
./scripts/micro/mc_probe > gpurun_out/p_mc_probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/p_pytest.log
timeout 300 python bench.py > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err
CMD="python bench.py --steps 5 --warmup 3 --phased-steps 2 --no-cpu-baseline"
$CMD > gpurun_out/p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p_launches.csv $CMD > gpurun_out/p_ncu1.log 2>&1
$CMD > gpurun_out/p_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_lamb_fused -s 20 -c 1 -o gpurun_out/p_lamb $CMD > gpurun_out/p_ncu2.log 2>&1
cat gpurun_out/p_mc_probe.txt gpurun_out/p_pytest.log gpurun_out/p_bench.json
tail -3 gpurun_out/p_ncu1.log gpurun_out/p_ncu2.log
