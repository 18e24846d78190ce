#!/bin/bash
# 1-GPU call: parity suite, bench, per-kernel check.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; python - <<'P'
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print({k: d[k] for k in ['ms_per_step','value','iterations']}, d['apply'], {k: d['roofline'][k] for k in ['achieved','frac','launch_ms']}, d['e2e']['ms_per_step'], d['cpu_baseline']['value'] if d['cpu_baseline'] else None, d['clocks'])
P
