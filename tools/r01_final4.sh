#!/bin/bash
# 4-GPU call: GPU tests (incl. 2/4-rank parity), weak scaling N=1,2,4 with the reference arm at N=1.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu4.log
python bench.py > gpurun_out/scale_n1.log 2>&1; echo "bench 1 rc=$?"
python bench.py --impl reference > gpurun_out/ref_n1.log 2>&1; echo "ref 1 rc=$?"; tail -1 gpurun_out/ref_n1.log | cut -c1-200
for W in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2955$W bench.py --gpus $W > gpurun_out/scale_n$W.log 2>&1; echo "bench $W rc=$?"; grep -iE "error" gpurun_out/scale_n$W.log | head -3
done
for W in 1 2 4; do python - $W <<'P'
import json,sys
W=sys.argv[1]
d=json.loads([l for l in open(f'gpurun_out/scale_n{W}.log') if l.startswith('{')][-1])
print(W, round(d['ms_per_step'],3), round(d['value'],1), d['iterations'], round(d['apply']['ms'],4), round(d['roofline']['frac'],3), round(d['e2e']['ms_per_step'],3), d['gpu_launches'], d['clocks'], (d.get('cpu_baseline') or {}).get('value'))
P
done
