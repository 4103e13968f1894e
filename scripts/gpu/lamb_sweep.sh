# k_lamb CTA-size sweep (build/variants/t*/libsp_round.so, built locally with
# -DSP_LAMB_THREADS=N), then one ncu --set full capture of the default build
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
LIB=paper_2106_10207_b200/lib/libsp_round.so
cp $LIB /tmp/default.so
for v in build/variants/t*; do
  cp $v/libsp_round.so $LIB
  for w in albert-large-fp16 albert-large-q8 albert-large-fp32; do
    timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-virtual-peers --workload $w > gpurun_out/sw_$(basename $v)_$w.json 2> gpurun_out/sw_$(basename $v)_$w.err
  done
done
cp /tmp/default.so $LIB
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lamb --launch-skip 5 -c 1 -o gpurun_out/ncu_lamb_r2a python bench.py --steps 3 --warmup 3 --phased-steps 1 --no-cpu-baseline --no-virtual-peers > gpurun_out/ncu_lamb_r2a.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_lamb_r2a.log
