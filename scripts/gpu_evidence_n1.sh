# Round-1 evidence on ONE B200: bench lines (default + other workloads + reference arm)
# and ncu launch list / full capture of the hot kernels.
export SP_SKIP_BUILD=1
mkdir -p gpurun_out/ev
python bench.py --steps 100 --warmup 5 > gpurun_out/ev/bench_n1.json 2> gpurun_out/ev/bench_n1.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_n1_reference.json 2>/dev/null
for w in resnet50-q8 albert-large-fp32 albert-large-q8 albert-base-fp32; do
  python bench.py --steps 100 --warmup 5 --no-cpu-baseline --workload $w > gpurun_out/ev/bench_n1_$w.json 2>/dev/null
done
python bench.py --steps 100 --warmup 5 --no-cpu-baseline --peers-per-gpu 8 > gpurun_out/ev/bench_n1_8virtualpeers.json 2>/dev/null
CMD="python scripts/profile_round.py --steps 3"
$CMD > gpurun_out/ev/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ev/launches_n1.csv $CMD > gpurun_out/ev/ncu_launch.log 2>&1
$CMD > gpurun_out/ev/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_lamb_fused|k_pack' -s 2 -c 2 \
    -o gpurun_out/ev/prof_n1 $CMD > gpurun_out/ev/ncu_full.log 2>&1
CMD8="python scripts/profile_round.py --steps 3 --peers 8"
$CMD8 > gpurun_out/ev/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_reduce' -s 1 -c 1 \
    -o gpurun_out/ev/prof_reduce_g8 $CMD8 > gpurun_out/ev/ncu_full_reduce.log 2>&1
ls -la gpurun_out/ev
