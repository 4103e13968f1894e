TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python -m pytest tests/test_round_gpu.py -x -q -k "shard" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_multigpu.py -x -q -k "sharded_lamb and not hybrid and not schedules" 2>&1 | tail -1
for N in 2 4; do for W in albert-large-fp16 albert-large-q8; do
  timeout 300 $TR --nproc-per-node $N --master-port $((29600+RANDOM%300)) bench.py --gpus $N --workload $W --no-cpu-baseline --phased-steps 5 > gpurun_out/g_n${N}_$W.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/g_n${N}_$W.json').read()); print('N=$N $W', d['round_us'], d['config']['lamb'][:9], {k:round(v*1e3,1) for k,v in d['kernel_ms'].items()})"
done; done
