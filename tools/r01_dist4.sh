#!/bin/bash
# 4-GPU call: distributed parity at 2 and 4 ranks, bench at N=2 and N=4.
mkdir -p gpurun_out
for W in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2953$W tests/dist_check.py > gpurun_out/dist_check_$W.log 2>&1; echo "dist_check $W rc=$?"
grep -E '^\{' gpurun_out/dist_check_$W.log | cut -c1-420; grep -E "Error|error" gpurun_out/dist_check_$W.log | head -5
done
for W in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2954$W bench.py --gpus $W --steps 30 --warmup 3 > gpurun_out/bench_n$W.log 2>&1; echo "bench $W rc=$?"; grep -E '^\{' gpurun_out/bench_n$W.log | cut -c1-300; grep -E "Error|error" gpurun_out/bench_n$W.log | head -5
done
