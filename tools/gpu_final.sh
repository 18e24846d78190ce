#!/bin/bash
# round-end evidence on one B200: pytest -m gpu, default bench line (+ cpu baselines, extra
# configs), the reference arm, per-kernel ncu launch list with DRAM bytes, ncu --set full of
# the interior solve
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench_n1.jsonl 2> gpurun_out/bench_n1.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_n1.jsonl 2> gpurun_out/bench_ref_n1.err; echo "ref rc $?"
PCG=1 NAPPLY=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/kernels.csv python tools/profile_apply.py > gpurun_out/ncu1.log 2>&1; echo "ncu list rc $?"
PCG=0 NAPPLY=3 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:interior_solve_kernel<\\(int\\)(0|3)," -s 2 -c 2 \
  -o gpurun_out/interior_full python tools/profile_apply.py > gpurun_out/ncu2.log 2>&1; echo "ncu full rc $?"
# the bench command's own launch list: the BDDC-PCG kernels (the setup kernels filtered out by name)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  -k "regex:^(interior_solve_kernel|iface_|spmv_dot|update_kernel|xpay_kernel|init_rho|dot_kernel|finalize_kernel|coarse_)" \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu3.log 2>&1; echo "ncu bench list rc $?"
