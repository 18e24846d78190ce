#!/bin/bash
# compare library variants (lib/libbddc_b200<V>.so) on the C2 bench line; restores the default
mkdir -p gpurun_out
cp paper_2410_14786_b200/lib/libbddc_b200.so /tmp/libdefault.so
for V in ${VARIANTS:-_w32 _w24 default}; do
  if [ "$V" = default ]; then cp /tmp/libdefault.so paper_2410_14786_b200/lib/libbddc_b200.so;
  else cp paper_2410_14786_b200/lib/libbddc_b200$V.so paper_2410_14786_b200/lib/libbddc_b200.so; fi
  timeout 300 python tools/gpu_check.py c2 > gpurun_out/check$V.log 2>&1 || echo "check $V failed"
  timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 20 > gpurun_out/bench$V.jsonl 2> gpurun_out/bench$V.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/bench$V.jsonl').read().strip().splitlines()[-1])
print('$V', 'ms', round(d['ms_per_step'],4), 'launch', round(d['roofline']['launch_ms'],4), 'frac', round(d['roofline']['frac'],3), 'apply', round(d['apply']['ms'],4), 'iters', d['iterations'])"
  tail -c 300 gpurun_out/check$V.log
done
cp /tmp/libdefault.so paper_2410_14786_b200/lib/libbddc_b200.so
