#!/bin/bash
# 2-GPU call: GPU parity suite; A/B of $VAR (N=1 x2 each, N=2 x1 each); 2-rank parity.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29538 tests/dist_check.py > gpurun_out/dist_check_2f.log 2>&1; echo "dist_check 2 rc=$?"
grep -E '^\{' gpurun_out/dist_check_2f.log | grep -c '"ok": true'; grep -E '"ok": false' gpurun_out/dist_check_2f.log | cut -c1-300
for V in 1 0 1 0; do
env $VAR=$V python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$V.log 2>&1
python - $V 1 <<'P'
import json,sys
d=json.loads([l for l in open(f'gpurun_out/ab_{sys.argv[1]}.log') if l.startswith('{')][-1])
print('N=1', sys.argv[1], round(d['ms_per_step'],3), d['iterations'], round(d['apply']['ms'],4), round(d['e2e']['ms_per_step'],3), d['gpu_launches'])
P
done
for V in 1 0; do
env $VAR=$V timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2957$V bench.py --gpus 2 --steps 30 --warmup 3 > gpurun_out/ab2_$V.log 2>&1
python - $V <<'P'
import json,sys
d=json.loads([l for l in open(f'gpurun_out/ab2_{sys.argv[1]}.log') if l.startswith('{')][-1])
print('N=2', sys.argv[1], round(d['ms_per_step'],3), d['iterations'], round(d['apply']['ms'],4), round(d['e2e']['ms_per_step'],3), d['gpu_launches'])
P
done
