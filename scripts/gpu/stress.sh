# repeated 1- and 2-GPU rounds (hang / race hunting): each run under its own timeout
mkdir -p gpurun_out/stress
export SP_SKIP_BUILD=1
O=gpurun_out/stress
for i in 1 2 3 4 5 6; do
  for w in albert-large-q8 albert-large-fp16; do
    timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + i)) \
      bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-virtual-peers --workload $w > $O/n2_${w}_$i.json 2> $O/n2_${w}_$i.err
    echo "n2 $w $i rc=$?" >> $O/rc.txt
  done
  timeout 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-virtual-peers > $O/n1_$i.json 2> $O/n1_$i.err
  echo "n1 $i rc=$?" >> $O/rc.txt
done
timeout 600 python -m pytest tests/test_round_gpu.py tests/test_multigpu.py -q --timeout 120 > $O/test.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
