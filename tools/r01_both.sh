#!/bin/bash
# 2-GPU call: GPU parity suite, N=1 bench, 2-rank parity, N=2 bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b_n1.log 2>&1; echo "bench 1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29538 tests/dist_check.py > gpurun_out/dist_check_2f.log 2>&1; echo "dist_check 2 rc=$?"
grep -E '^\{' gpurun_out/dist_check_2f.log | grep -c '"ok": true'; grep -E '"ok": false' gpurun_out/dist_check_2f.log | cut -c1-400; grep -iE "error|trap" gpurun_out/dist_check_2f.log | head -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --steps 30 --warmup 3 > gpurun_out/b_n2.log 2>&1; echo "bench 2 rc=$?"
for W in n1 n2; do python - $W <<'P'
import json,sys
W=sys.argv[1]
d=json.loads([l for l in open(f'gpurun_out/b_{W}.log') if l.startswith('{')][-1])
print(W, round(d['ms_per_step'],3), round(d['value'],1), d['iterations'], round(d['apply']['ms'],4), round(d['roofline']['launch_ms'],4), round(d['e2e']['ms_per_step'],3), d['gpu_launches'], d['clocks']['sm_mhz'])
P
done
