set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_round_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/u_pytest1.log
timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -3 > gpurun_out/u_pytest4.log
for N in 2 4; do
  for W in albert-large-fp16 albert-large-fp32 albert-large-q8; do
    timeout 300 $TR --nproc-per-node $N --master-port $((29500+N)) bench.py --gpus $N --workload $W --no-cpu-baseline > gpurun_out/u_n${N}_$W.json 2> gpurun_out/u_n${N}_$W.err
  done
done
cat gpurun_out/u_pytest1.log gpurun_out/u_pytest4.log
for f in gpurun_out/u_n*.json; do python -c "
import json; d=json.loads(open('$f').read()); rr=d.get('round_roofline') or {}; print('$f', d.get('round_us'), rr.get('frac'), {k:round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; done
