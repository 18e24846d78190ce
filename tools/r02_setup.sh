#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_setup.py -q -x > gpurun_out/pytest_setup.log 2>&1; echo "setup tests rc $?"
tail -30 gpurun_out/pytest_setup.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc $?"
tail -5 gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.jsonl').read().strip().splitlines()[-1])
print('c2 ms', d['ms_per_step'], 'setup', d['setup_seconds'], 'frac', d['roofline']['frac'])
for k,e in (d.get('extra_configs') or {}).items(): print(k, 'ms', e['ms_per_step'], 'it', e['iterations'], 'setup', e['setup_seconds'])
"
