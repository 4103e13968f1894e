export SP_SKIP_BUILD=1
N=$(nvidia-smi -L | wc -l)
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 3"
run() { echo "$* : $(env "$@" timeout 300 $T 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['round_us'])")"; }
run SP_SEGMENTS=1 SP_XCHG_PER_SM=8
run SP_SEGMENTS=1 SP_XCHG_PER_SM=4
run SP_SEGMENTS=1 SP_XCHG_PER_SM=2
for K in 2 4; do for G in 148 444; do for X in 2 4; do
run SP_SEGMENTS=$K SP_SEG_LAMB_GRID=$G SP_XCHG_PER_SM=$X
done; done; done
