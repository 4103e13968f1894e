# final 4-GPU validation: the whole GPU suite (incl. multi-GPU parity), N=2 and N=4 headline bench
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/z_pytest.log
timeout 300 $TR --nproc-per-node 2 --master-port 29602 bench.py --gpus 2 > gpurun_out/z_n2.json 2> gpurun_out/z_n2.err
timeout 300 $TR --nproc-per-node 4 --master-port 29604 bench.py --gpus 4 > gpurun_out/z_n4.json 2> gpurun_out/z_n4.err
timeout 300 $TR --nproc-per-node 4 --master-port 29605 bench.py --gpus 4 --impl reference > gpurun_out/z_n4_ref.json 2> gpurun_out/z_n4_ref.err
cat gpurun_out/z_pytest.log
for f in gpurun_out/z_n2.json gpurun_out/z_n4.json gpurun_out/z_n4_ref.json; do python -c "
import json; d=json.loads(open('$f').read()); print('$f', d.get('round_us'), d.get('value'), (d.get('round_roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), d.get('clocks'))"; done
