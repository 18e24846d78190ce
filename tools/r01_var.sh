#!/bin/bash
# 1-GPU call: N=1 bench repeated (variance check).
mkdir -p gpurun_out
for i in 1 2 3 4 5; do python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/v_$i.log 2>&1
python - $i <<'P'
import json,sys
d=json.loads([l for l in open(f'gpurun_out/v_{sys.argv[1]}.log') if l.startswith('{')][-1])
print(sys.argv[1], round(d['ms_per_step'],3), round(d['apply']['ms'],4), round(d['e2e']['ms_per_step'],3), d['clocks'])
P
done
