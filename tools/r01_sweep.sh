#!/bin/bash
# 1-GPU sweep of an env knob: bench N=1 (steps 20) per value in $VALS for $VAR.
mkdir -p gpurun_out
for V in $VALS; do
env $VAR=$V python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/sw_$V.log 2>&1
python - $V <<'P'
import json,sys
d=json.loads([l for l in open(f'gpurun_out/sw_{sys.argv[1]}.log') if l.startswith('{')][-1])
print(sys.argv[1], round(d['ms_per_step'],3), d['iterations'], round(d['apply']['ms'],4), round(d['roofline']['launch_ms'],4))
P
done
