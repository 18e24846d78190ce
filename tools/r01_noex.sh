#!/bin/bash
mkdir -p gpurun_out
for E in 1 0; do
BDDC_NO_EXCHANGE=$E timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954$E bench.py --gpus 2 --steps 30 --warmup 3 > gpurun_out/bench_noex$E.log 2>&1; echo "noex=$E rc=$?"
grep -E '^\{' gpurun_out/bench_noex$E.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['iterations'], round(d['apply']['ms'],4), d['gpu_launches'])"
done
python bench.py --steps 30 --warmup 3 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N=1', round(d['ms_per_step'],3), d['iterations'], round(d['apply']['ms'],4), d['gpu_launches'])"
