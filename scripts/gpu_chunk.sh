TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do for C in 4096 8192 16384 32768; do
  SP_LAMB_CHUNK=$C timeout 300 $TR --nproc-per-node $N --master-port $((29600+RANDOM%300)) bench.py --gpus $N --no-cpu-baseline --phased-steps 3 > gpurun_out/c_n${N}_$C.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/c_n${N}_$C.json').read()); print('N=$N chunk=$C', d['round_us'])"
done; done
