TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
SP_PUSH_CE=1 timeout 300 $TR --nproc-per-node 4 --master-port 29655 tests/mp_round_check.py --wire fp16 --shard-lamb 2>/dev/null | tail -1 | cut -c1-60
SP_PUSH_CE=1 timeout 300 $TR --nproc-per-node 2 --master-port 29656 tests/mp_round_check.py --wire q8 --shard-lamb 2>/dev/null | tail -1 | cut -c1-60
for N in 2 4; do for E in 0 1; do
  SP_PUSH_CE=$E timeout 300 $TR --nproc-per-node $N --master-port $((29600+RANDOM%300)) bench.py --gpus $N --no-cpu-baseline --phased-steps 3 > gpurun_out/e_n${N}_$E.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/e_n${N}_$E.json').read()); print('N=$N ce=$E', d['round_us'])"
  SP_PUSH_CE=$E timeout 300 $TR --nproc-per-node $N --master-port $((29600+RANDOM%300)) bench.py --gpus $N --no-cpu-baseline --phased-steps 3 --workload sweep --params 268435456 --wire fp16 --steps 10 > gpurun_out/e_n${N}_268m_$E.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/e_n${N}_268m_$E.json').read()); print('N=$N 268M ce=$E', d['round_us'])"
done; done
