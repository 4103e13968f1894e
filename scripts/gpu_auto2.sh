# --lamb auto end to end on 2 GPUs: uniform (sharded) and dominant-owner fleets (replicated)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for W in albert-large-fp16 het8c-fp16 het4b-fp32; do
  timeout 300 $TR --master-port $((29600+RANDOM%300)) bench.py --gpus 2 --workload $W --no-cpu-baseline > gpurun_out/a_n2_$W.json 2> gpurun_out/a_n2_$W.err
  python -c "import json; d=json.loads(open('gpurun_out/a_n2_$W.json').read()); print('N=2 $W', d['round_us'], d['config']['lamb'][:10], d['round_roofline']['frac'], d['roofline']['kernel'], d['roofline']['frac'], d['gpu_launches'])"
done
