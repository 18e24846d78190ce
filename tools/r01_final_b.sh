#!/bin/bash
# Final measurement call B (1 GPU): ncu --set full of the two interior-solve launches of one apply.
mkdir -p gpurun_out
PCG=0 NAPPLY=3 python tools/profile_apply.py > gpurun_out/plain2.log 2>&1 && \
PCG=0 NAPPLY=3 ncu --set full --clock-control none --import-source on -k regex:interior_solve -s 2 -c 2 \
    -o gpurun_out/solve_c2 python tools/profile_apply.py > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_full.log
