set -x
nvidia-smi topo -m > gpurun_out/q_topo.txt 2>&1
nvidia-smi nvlink -s -i 0 > gpurun_out/q_nvlink.txt 2>&1
./scripts/micro/p2p_bw 16 > gpurun_out/q_p2p2_16.txt 2>&1
./scripts/micro/p2p_bw 256 > gpurun_out/q_p2p2_256.txt 2>&1
cat gpurun_out/q_topo.txt gpurun_out/q_p2p2_16.txt gpurun_out/q_p2p2_256.txt
