set -x
python tools/profile_apply.py > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_apply.py > gpurun_out/ncu1.log 2>&1
PCG=0 NAPPLY=3 python tools/profile_apply.py > gpurun_out/plain2.log 2>&1 && \
PCG=0 NAPPLY=3 ncu --set full --clock-control none --import-source on -k regex:interior_solve -s 2 -c 1 -o gpurun_out/solve_c2 python tools/profile_apply.py > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu2.log
