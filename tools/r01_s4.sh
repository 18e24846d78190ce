#!/bin/bash
# 4-GPU call: 4-rank parity + weak scaling N=1,2,4 (bench lines).
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29538 tests/dist_check.py > gpurun_out/dist_check_4.log 2>&1; echo "dist_check 4 rc=$?"
grep -E '^\{' gpurun_out/dist_check_4.log | grep -c '"ok": true'; grep -E '"ok": false' gpurun_out/dist_check_4.log | cut -c1-300
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/scale_n1.log 2>&1; echo "bench 1 rc=$?"
for W in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2955$W bench.py --gpus $W --steps 30 --warmup 3 > gpurun_out/scale_n$W.log 2>&1; echo "bench $W rc=$?"
done
for W in 1 2 4; do python - $W <<'P'
import json,sys
W=sys.argv[1]
d=json.loads([l for l in open(f'gpurun_out/scale_n{W}.log') if l.startswith('{')][-1])
print(W, round(d['ms_per_step'],3), round(d['value'],1), d['iterations'], round(d['apply']['ms'],4), round(d['e2e']['ms_per_step'],3), d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
P
done
