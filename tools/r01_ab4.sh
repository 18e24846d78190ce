#!/bin/bash
# 4-GPU call: A/B of $VAR at N=4 and N=1 (bench lines).
mkdir -p gpurun_out
for V in 1 0 1 0; do
env $VAR=$V timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2958$V bench.py --gpus 4 --steps 30 --warmup 3 > gpurun_out/ab4_$V.log 2>&1
python - $V <<'P'
import json,sys
d=json.loads([l for l in open(f'gpurun_out/ab4_{sys.argv[1]}.log') if l.startswith('{')][-1])
print('N=4', sys.argv[1], round(d['ms_per_step'],3), round(d['apply']['ms'],4), round(d['e2e']['ms_per_step'],3))
P
done
for V in 1 0; do
env $VAR=$V python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ab1_$V.log 2>&1
python - $V <<'P'
import json,sys
d=json.loads([l for l in open(f'gpurun_out/ab1_{sys.argv[1]}.log') if l.startswith('{')][-1])
print('N=1', sys.argv[1], round(d['ms_per_step'],3), round(d['apply']['ms'],4), round(d['e2e']['ms_per_step'],3))
P
done
