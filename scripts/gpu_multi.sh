# N=2 and N=4 over NVLink: multi-GPU parity tests, headline + fleet workloads, N=2 sweep, reference arm
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -3 > gpurun_out/m_pytest.log
for N in 2 4; do
  for W in albert-large-fp16 albert-large-fp32 albert-large-q8 resnet50-q8 het8c-fp16 het4b-fp32; do
    timeout 300 $TR --nproc-per-node $N --master-port $((29500+N)) bench.py --gpus $N --workload $W --no-cpu-baseline > gpurun_out/m_n${N}_$W.json 2> gpurun_out/m_n${N}_$W.err
  done
done
timeout 300 $TR --nproc-per-node 4 --master-port 29512 bench.py --gpus 4 --impl reference > gpurun_out/m_n4_reference.json 2> gpurun_out/m_n4_reference.err
rm -f gpurun_out/m_sweep_n2.jsonl
timeout 1500 python scripts/sweep.py --gpus 2 --out gpurun_out/m_sweep_n2.jsonl
cat gpurun_out/m_pytest.log
for f in gpurun_out/m_n*.json; do python -c "
import json; d=json.loads(open('$f').read()); rr=d.get('round_roofline') or {}; print('$f', d.get('round_us'), d.get('value'), rr.get('frac'), rr.get('frac_overlap'), (d.get('e2e') or {}).get('value'))"; done
