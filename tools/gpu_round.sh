#!/bin/bash
# single-GPU round check: parity suite (minus distributed), bench line, launch list
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_distributed.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --steps 20 ${BENCH_ARGS} > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc $?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.jsonl').read().strip().splitlines()[-1])
print('c2 ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'setup', round(d['setup_seconds'],3), 'frac', round(d['roofline']['frac'],4), 'apply', round(d['apply']['ms'],4))
for k,e in (d.get('extra_configs') or {}).items(): print(k, 'ms', round(e['ms_per_step'],3), 'it', e['iterations'], 'setup', round(e['setup_seconds'],3))
"
PCG=1 NAPPLY=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/kernels.csv python tools/profile_apply.py > gpurun_out/ncu1.log 2>&1; echo "ncu rc $?"
