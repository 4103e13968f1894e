# round-end style check on one B200: all GPU tests, smoke, the default bench
# and the reference arm, the ncu launch list and one full capture of k_lamb
mkdir -p gpurun_out/full
export SP_SKIP_BUILD=1
O=gpurun_out/full
nvidia-smi -L > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > $O/test.log 2>&1; echo "pytest rc=$?" >> $O/test.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lamb --launch-skip 5 -c 1 -o $O/ncu_lamb python bench.py --steps 3 --warmup 3 --phased-steps 1 --no-cpu-baseline --no-virtual-peers > $O/ncu_full.log 2>&1
