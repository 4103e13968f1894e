# ncu evidence for the round: launch list (per-kernel device times) and one
# full capture of each hot kernel. Run under gpurun on ONE GPU.
set -x
export SP_SKIP_BUILD=1
mkdir -p gpurun_out
CMD="python scripts/profile_round.py --steps 3"
$CMD > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_lamb|k_reduce|k_pack' -s 6 -c 4 \
    -o gpurun_out/prof_round $CMD > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; cat gpurun_out/bench_r1b.json
