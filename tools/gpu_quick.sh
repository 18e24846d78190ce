#!/bin/bash
# dev helper: run the GPU probe config by config with short timeouts
python -c "import __graft_entry__ as g; g.smoke()" || exit 1
for c in k4m8 c1 c2; do
  timeout ${T:-90} python tools/gpu_check.py $c || echo "FAILED/TIMEOUT $c"
done
