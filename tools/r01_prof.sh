#!/bin/bash
# Profiling call: bench (N=1, full), ncu launch list of the bench, ncu --set full of the interior solve.
mkdir -p gpurun_out
python bench.py --steps 30 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
PCG=0 NAPPLY=3 python tools/profile_apply.py > gpurun_out/plain2.log 2>&1 && \
PCG=0 NAPPLY=3 ncu --set full --clock-control none --import-source on -k regex:interior_solve -s 2 -c 2 \
    -o gpurun_out/solve_c2 python tools/profile_apply.py > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -1 gpurun_out/ncu_full.log
