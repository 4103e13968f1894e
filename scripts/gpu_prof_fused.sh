set -x
export SP_SKIP_BUILD=1
CMD="python scripts/profile_round.py --steps 3"
$CMD > gpurun_out/plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_round_fused -s 1 -c 1 -o gpurun_out/prof_fused $CMD > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/ncu_fused.log
