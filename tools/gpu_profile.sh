#!/bin/bash
# round-2 profiling recipe: parity probe, per-kernel DRAM bytes of a C2 solve, full capture of the interior solve
mkdir -p gpurun_out
timeout 600 python tools/plain_probe.py > gpurun_out/plain_probe.log 2>&1; echo "probe rc $?"
PCG=1 NAPPLY=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file gpurun_out/r02_kernels.csv python tools/profile_apply.py > gpurun_out/r02_ncu1.log 2>&1; echo "ncu1 rc $?"
PCG=0 NAPPLY=3 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:interior_solve_kernel<\\(int\\)(0|3)," -s 2 -c 2 \
  -o gpurun_out/r02_solve python tools/profile_apply.py > gpurun_out/r02_ncu2.log 2>&1; echo "ncu2 rc $?"
