# build/variants/w*/libsp_round.so (k_lamb compile-time configurations and
# diagnostic builds, built locally): N=1 ALBERT-large fp16 bench, 2
# interleaved repetitions per variant
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
LIB=paper_2106_10207_b200/lib/libsp_round.so
cp $LIB /tmp/default.so
for rep in 1 2; do
  for v in build/variants/w*; do
    cp $v/libsp_round.so $LIB
    timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-virtual-peers > gpurun_out/va_$(basename $v)_r$rep.json 2> gpurun_out/va_$(basename $v)_r$rep.err
  done
done
cp /tmp/default.so $LIB
