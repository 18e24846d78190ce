#!/bin/bash
cp paper_2410_14786_b200/lib/libbddc_b200.so /tmp/libnew.so
for V in new old new old; do
  cp /tmp/lib$V.so paper_2410_14786_b200/lib/libbddc_b200.so 2>/dev/null || cp paper_2410_14786_b200/lib/libbddc_b200_old.so paper_2410_14786_b200/lib/libbddc_b200.so
  [ $V = old ] && cp paper_2410_14786_b200/lib/libbddc_b200_old.so paper_2410_14786_b200/lib/libbddc_b200.so
  echo "== $V"; timeout 300 python bench.py --config c4 --no-extra --no-cpu-baseline --steps 5 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['clocks'])"
done
cp /tmp/libnew.so paper_2410_14786_b200/lib/libbddc_b200.so
