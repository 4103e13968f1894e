TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
for W in 1.0 0.5 0.25 0.1; do
for X in 8 4; do
  SP_XCHG_PER_SM=$X SP_PACK_LOCAL_WEIGHT=$W timeout 300 $TR --nproc-per-node $N --master-port $((29600+RANDOM%300)) bench.py --gpus $N --no-cpu-baseline --phased-steps 5 > gpurun_out/w_n${N}_${W}_$X.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/w_n${N}_${W}_$X.json').read()); print('N=$N w=$W xps=$X', d['round_us'], {k:round(v*1e3,1) for k,v in d['kernel_ms'].items() if k in ('pack_ms','barrier_a_ms')})"
done; done; done
