# (knobs updated: the chain is the default, SP_SHARD_FUSED=1 selects the one-kernel variant)
# one-kernel sharded LAMB: parity (1 and 4 GPUs), then N=2/N=4 bench vs the kernel chain
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_round_gpu.py -x -q -k "shard" 2>&1 | tail -3 > gpurun_out/s_pytest1.log
timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "shard" 2>&1 | tail -3 > gpurun_out/s_pytest4.log
for N in 2 4; do
  for W in albert-large-fp16 albert-large-fp32 albert-large-q8; do
    SP_SHARD_FUSED=1 timeout 300 $TR --nproc-per-node $N --master-port $((29500+N)) bench.py --gpus $N --workload $W --no-cpu-baseline > gpurun_out/s_n${N}_$W.json 2> gpurun_out/s_n${N}_$W.err
    SP_SHARD_FUSED=1 SP_SHARD_LAG=600 timeout 300 $TR --nproc-per-node $N --master-port $((29510+N)) bench.py --gpus $N --workload $W --no-cpu-baseline > gpurun_out/s_n${N}_${W}_lag600.json 2> /dev/null
    SP_SHARD_FUSED=0 timeout 300 $TR --nproc-per-node $N --master-port $((29520+N)) bench.py --gpus $N --workload $W --no-cpu-baseline > gpurun_out/s_n${N}_${W}_chain.json 2> /dev/null
  done
  SP_LAMB_CHUNK=4096 timeout 300 $TR --nproc-per-node $N --master-port $((29530+N)) bench.py --gpus $N --no-cpu-baseline > gpurun_out/s_n${N}_c4096.json 2> /dev/null
  SP_LAMB_CHUNK=16384 timeout 300 $TR --nproc-per-node $N --master-port $((29540+N)) bench.py --gpus $N --no-cpu-baseline > gpurun_out/s_n${N}_c16384.json 2> /dev/null
  timeout 300 $TR --nproc-per-node $N --master-port $((29550+N)) bench.py --gpus $N --workload sweep --params 268435456 --wire fp16 --steps 10 --no-cpu-baseline > gpurun_out/s_n${N}_268m.json 2> /dev/null
done
cat gpurun_out/s_pytest1.log gpurun_out/s_pytest4.log
for f in gpurun_out/s_n*.json; do python -c "
import json; d=json.loads(open('$f').read()); rr=d.get('round_roofline') or {}; print('$f', d.get('round_us'), rr.get('frac'), {k:round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; done
