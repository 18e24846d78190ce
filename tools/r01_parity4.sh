#!/bin/bash
# 4-GPU call: full GPU test suite, distributed parity at 2 and 4 ranks (incl. C3 at 4), C3 bench point.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 tests/dist_check.py > gpurun_out/dist_check_2.log 2>&1; echo "dist_check 2 rc=$?"
grep -E '^\{' gpurun_out/dist_check_2.log | grep -c '"ok": true'; grep -E '"ok": false' gpurun_out/dist_check_2.log | cut -c1-500
DIST_CHECK_C3=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 tests/dist_check.py > gpurun_out/dist_check_4.log 2>&1; echo "dist_check 4 rc=$?"
grep -E '^\{' gpurun_out/dist_check_4.log | grep -c '"ok": true'; grep -E '"ok": false' gpurun_out/dist_check_4.log | cut -c1-500; grep -iE "error" gpurun_out/dist_check_4.log | head -3
grep -E '"config": "c3"' gpurun_out/dist_check_4.log | cut -c1-400
