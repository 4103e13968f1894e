# (knobs updated: the chain is the default, SP_SHARD_FUSED=1 selects the one-kernel variant)
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_multigpu.py -x -q -k "ragged_owners or one_kernel" 2>&1 | tail -3 > gpurun_out/t_pytest4.log
for V in 0 64 600 chain; do
  E="SP_SHARD_FUSED=1 SP_SHARD_LAG=$V"; [ $V = chain ] && E="SP_SHARD_FUSED=0"
  env $E timeout 300 $TR --nproc-per-node 4 --master-port $((29600+RANDOM%100)) bench.py --gpus 4 --no-cpu-baseline --phased-steps 5 > gpurun_out/t_n4_$V.json 2> /dev/null
  env $E timeout 300 $TR --nproc-per-node 4 --master-port $((29700+RANDOM%100)) bench.py --gpus 4 --no-cpu-baseline --phased-steps 5 --workload sweep --params 268435456 --wire fp16 --steps 10 > gpurun_out/t_n4_268m_$V.json 2> /dev/null
done
cat gpurun_out/t_pytest4.log
for f in gpurun_out/t_n*.json; do python -c "
import json; d=json.loads(open('$f').read()); print('$f', d.get('round_us'), {k:round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; done
