# final check on two B200s: every GPU test (multi-GPU ones at 2 GPUs), smoke,
# and repeated 1- and 2-GPU rounds
mkdir -p gpurun_out/final2
export SP_SKIP_BUILD=1
O=gpurun_out/final2
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > $O/test.log 2>&1; echo "pytest rc=$?" >> $O/test.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for i in 1 2 3; do
  for w in albert-large-q8 albert-large-fp16 resnet50-q8; do
    timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + i)) \
      bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-virtual-peers --workload $w > $O/n2_${w}_$i.json 2> $O/n2_${w}_$i.err
    echo "n2 $w $i rc=$?" >> $O/rc.txt
  done
done
