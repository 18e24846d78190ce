#!/bin/bash
# 1-GPU call: parity subset, bench x2, ncu launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/pytest_parity.log
for i in 1 2; do python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/n1.log 2>&1
python - <<'P'
import json
d=json.loads([l for l in open('gpurun_out/n1.log') if l.startswith('{')][-1])
print(round(d['ms_per_step'],3), d['iterations'], round(d['apply']['ms'],4), round(d['roofline']['launch_ms'],4), round(d['e2e']['ms_per_step'],3), d['gpu_launches'], d['clocks']['sm_mhz'])
P
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
