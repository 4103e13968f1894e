# 2 and 4 GPUs on one box: multi-GPU parity tests, then ALBERT-large with the
# LAMB mode chosen by the plan (auto) and with each mode forced
mkdir -p gpurun_out/mm
export SP_SKIP_BUILD=1
O=gpurun_out/mm
timeout 900 python -m pytest tests/test_multigpu.py -q --timeout 600 > $O/test_n4.log 2>&1; echo "pytest rc=$?" >> $O/test_n4.log
for N in 2 4; do
  if [ $N = 2 ]; then export CUDA_VISIBLE_DEVICES=0,1; else unset CUDA_VISIBLE_DEVICES; fi
  for w in albert-large-fp16 albert-large-q8 het8c-fp16; do
    for mode in auto replicated sharded; do
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 \
        bench.py --gpus $N --steps 30 --warmup 5 --no-cpu-baseline --workload $w --lamb $mode > $O/n${N}_${w}_$mode.json 2> $O/n${N}_${w}_$mode.err
    done
  done
done
