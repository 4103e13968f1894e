# N=1: LP-planned fleets (BASELINE configs 1, 4) and the size x wire sweep (config 5)
set -x
timeout 300 python bench.py > gpurun_out/b_default.json 2> gpurun_out/b_default.err
timeout 300 python bench.py --workload het8c-fp16 > gpurun_out/b_het8c_n1.json 2> gpurun_out/b_het8c_n1.err
timeout 300 python bench.py --workload het4b-fp32 > gpurun_out/b_het4b_n1.json 2> gpurun_out/b_het4b_n1.err
rm -f gpurun_out/sweep_n1.jsonl
timeout 1500 python scripts/sweep.py --gpus 1 --out gpurun_out/sweep_n1.jsonl
cat gpurun_out/b_default.json gpurun_out/b_het8c_n1.json gpurun_out/b_het4b_n1.json
tail -3 gpurun_out/*.err
