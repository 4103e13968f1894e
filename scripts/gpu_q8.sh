# q8 wire: parity tests, bench, launch list and a full capture of pack + LAMB.
export SP_SKIP_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --workload albert-large-q8 --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 10 > gpurun_out/bench_q8.json 2>gpurun_out/bench_q8.err
python -c "import json; d=json.load(open('gpurun_out/bench_q8.json')); print(d['round_us'], d['kernel_ms'], d['roofline'])"
CMD="python scripts/profile_round.py --wire q8 --steps 3"
$CMD > gpurun_out/plain_q8.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_q8.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_lamb|k_pack' -s 2 -c 2 \
    -o gpurun_out/prof_q8 $CMD > gpurun_out/ncu_q8.log 2>&1
tail -2 gpurun_out/ncu_q8.log
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --phased-steps 10 > gpurun_out/bench_fp16.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_fp16.json')); print('fp16', d['round_us'], d['kernel_ms'])"
