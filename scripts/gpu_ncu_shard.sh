# ncu evidence for the N>1 kernels, run at world 1 (ncu never wraps a multi-rank command):
# sharded pass 1 / pass 2 + push over an ALBERT-large-sized owned range, pack + reduce with 2 virtual peers
CMD="python bench.py --steps 3 --warmup 3 --phased-steps 1 --no-cpu-baseline --lamb sharded --peers-per-gpu 2"
$CMD > gpurun_out/n_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_lamb_moments_shard|k_lamb_update_push_trust|k_pack_fp16|k_reduce_fp16" -s 8 -c 4 -o gpurun_out/n_shard $CMD > gpurun_out/n_ncu.log 2>&1
tail -3 gpurun_out/n_ncu.log
