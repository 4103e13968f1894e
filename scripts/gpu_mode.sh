TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
for W in het8c-fp16 het4b-fp32; do
for M in sharded replicated; do
  timeout 300 $TR --nproc-per-node $N --master-port $((29600+RANDOM%300)) bench.py --gpus $N --workload $W --lamb $M --no-cpu-baseline --phased-steps 5 > gpurun_out/v_n${N}_${W}_$M.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/v_n${N}_${W}_$M.json').read()); print('N=$N $W $M', d['round_us'], d['round_roofline']['t_roof_us'])"
done; done; done
