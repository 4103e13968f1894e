TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python -m pytest tests/test_round_gpu.py -x -q 2>&1 | tail -1
timeout 600 python -m pytest tests/test_multigpu.py -x -q -k "sharded or uniform or nonuniform" 2>&1 | tail -1
for W in albert-large-fp16 albert-large-fp32; do for E in 0 1; do
  V=""; [ $E = 0 ] && V="SP_NO_FUSED_REDUCE=1"
  env $V SP_X=1 timeout 300 $TR --nproc-per-node 2 --master-port $((29600+RANDOM%300)) bench.py --gpus 2 --workload $W --no-cpu-baseline --phased-steps 3 > gpurun_out/r_$W_$E.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/r_$W_$E.json').read()); print('N=2 $W fused_reduce=$E', d['round_us'])"
done; done
