#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for H in 1 0; do BDDC_HARMONIC=$H python bench.py --no-cpu-baseline > gpurun_out/bench_h$H.log 2>&1; echo "N=1 harmonic=$H rc=$?"
grep -E '^\{' gpurun_out/bench_h$H.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['iterations'], round(d['apply']['ms'],4), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3), round(d['e2e']['ms_per_step'],3))"; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 > gpurun_out/bench_n2.log 2>&1; echo "N=2 rc=$?"
grep -E '^\{' gpurun_out/bench_n2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['iterations'], round(d['apply']['ms'],4), round(d['roofline']['frac'],3), round(d['e2e']['ms_per_step'],3))"
