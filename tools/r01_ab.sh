#!/bin/bash
# 1-GPU A/B of an env toggle: bench N=1 alternating $VAR=0/1 twice, then a launch list.
mkdir -p gpurun_out
for V in 1 0 1 0; do
env $VAR=$V python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$V.log 2>&1
python - $V <<'P'
import json,sys
d=json.loads([l for l in open(f'gpurun_out/ab_{sys.argv[1]}.log') if l.startswith('{')][-1])
print(sys.argv[1], round(d['ms_per_step'],3), d['iterations'], round(d['apply']['ms'],4), round(d['e2e']['ms_per_step'],3), d['gpu_launches'])
P
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
