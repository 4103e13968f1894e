# N=2 and N=4 over NVLink: headline workloads, LP fleets, sweep subset, multi-GPU tests
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_multigpu.py tests/test_world8.py -x -q 2>&1 | tail -5 > gpurun_out/n4_pytest.log
for N in 2 4; do
  for W in albert-large-fp16 albert-large-fp32 albert-large-q8 resnet50-q8 het8c-fp16; do
    timeout 300 $TR --nproc-per-node $N --master-port $((29500+N)) bench.py --gpus $N --workload $W > gpurun_out/n${N}_$W.json 2> gpurun_out/n${N}_$W.err
  done
done
timeout 300 $TR --nproc-per-node 4 --master-port 29510 bench.py --gpus 4 --workload het4b-fp32 > gpurun_out/n4_het4b-fp32.json 2> gpurun_out/n4_het4b-fp32.err
timeout 300 $TR --nproc-per-node 4 --master-port 29511 bench.py --gpus 4 --lamb replicated > gpurun_out/n4_albert-large-fp16-replicated.json 2> gpurun_out/n4_replicated.err
timeout 300 $TR --nproc-per-node 4 --master-port 29512 bench.py --gpus 4 --impl reference > gpurun_out/n4_reference.json 2> gpurun_out/n4_reference.err
rm -f gpurun_out/sweep_n4.jsonl gpurun_out/sweep_n2.jsonl
timeout 1200 python scripts/sweep.py --gpus 4 --out gpurun_out/sweep_n4.jsonl
timeout 900 python scripts/sweep.py --gpus 2 --out gpurun_out/sweep_n2.jsonl --sizes 4194304,67108864,1073741824
cat gpurun_out/n4_pytest.log
for f in gpurun_out/n[24]_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d.get('round_us'), d.get('value'), (d.get('round_roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'))"; done
