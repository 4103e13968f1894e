# multi-GPU checks on one box (run with gpurun --gpus N): the multi-rank
# parity tests, then the N-GPU bench (torchrun, one process per GPU)
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests/test_multigpu.py -q --timeout 600 > gpurun_out/mg_test_n$N.log 2>&1
echo "pytest rc=$?" >> gpurun_out/mg_test_n$N.log
for w in albert-large-fp16 het8c-fp16 albert-large-q8 resnet50-q8; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 30 --warmup 5 --no-cpu-baseline --workload $w > gpurun_out/mg_n${N}_$w.json 2> gpurun_out/mg_n${N}_$w.err
done
