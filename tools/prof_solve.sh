PCG=0 NAPPLY=3 python tools/profile_apply.py > gpurun_out/plain2.log 2>&1 && \
PCG=0 NAPPLY=3 ncu --set full --clock-control none --import-source on -k regex:interior_solve -s 2 -c 1 -o gpurun_out/solve_v4 python tools/profile_apply.py > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu2.log
