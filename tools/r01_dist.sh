#!/bin/bash
# 2-GPU call: distributed parity driver, bench at N=2, then the GPU test suite.
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tests/dist_check.py > gpurun_out/dist_check.log 2>&1; echo "dist_check rc=$?"
grep -E '^\{' gpurun_out/dist_check.log | cut -c1-600; grep -E "Error|error" gpurun_out/dist_check.log | head -5
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 30 --warmup 3 > gpurun_out/bench_n2.log 2>&1; echo "bench2 rc=$?"; grep -E '^\{' gpurun_out/bench_n2.log | cut -c1-2500; grep -E "Error|error" gpurun_out/bench_n2.log | head -5
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu2.log
