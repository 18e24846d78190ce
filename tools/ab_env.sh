#!/bin/bash
# A/B of environment variants on one bench config, interleaved (VARIANTS with '+'-joined envs,
# CFGS, ROUNDS); device ms and e2e ms per line
mkdir -p gpurun_out
for rnd in $(seq 1 ${ROUNDS:-3}); do
for v in ${VARIANTS:-default}; do
for cfg in ${CFGS:-c2}; do
  if [ "$v" = default ]; then envs=""; else envs="${v//+/ }"; fi
  env $envs timeout 600 python bench.py --no-cpu-baseline --no-extra --steps ${STEPS:-20} --config $cfg > gpurun_out/abe.jsonl 2>gpurun_out/abe.err
  python -c "
import json; d=json.loads(open('gpurun_out/abe.jsonl').read().strip().splitlines()[-1])
print('$rnd $v $cfg ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'it', d['iterations'])
" || tail -5 gpurun_out/abe.err
done; done; done
