#!/bin/bash
# 2-GPU call: GPU tests, bench N=1 with/without graphs, dist parity, bench N=2 with/without graphs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for G in 1 0; do
BDDC_GRAPH=$G python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g$G.log 2>&1; echo "N=1 graph=$G rc=$?"
grep -E '^\{' gpurun_out/bench_g$G.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['iterations'], round(d['apply']['ms'],4), round(d['roofline']['launch_ms'],4), round(d['e2e']['ms_per_step'],3), d['gpu_launches'])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tests/dist_check.py > gpurun_out/dist_check_g.log 2>&1; echo "dist_check rc=$?"
grep -E '^\{' gpurun_out/dist_check_g.log | grep -c '"ok": true'; grep -iE "error" gpurun_out/dist_check_g.log | head -3
for G in 1 0; do
BDDC_GRAPH=$G timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2955$G bench.py --gpus 2 --steps 30 --warmup 3 > gpurun_out/bench_n2_g$G.log 2>&1; echo "N=2 graph=$G rc=$?"; grep -iE "error" gpurun_out/bench_n2_g$G.log | head -3
grep -E '^\{' gpurun_out/bench_n2_g$G.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['iterations'], round(d['apply']['ms'],4), round(d['e2e']['ms_per_step'],3), d['gpu_launches'])"
done
