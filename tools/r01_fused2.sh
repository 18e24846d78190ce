#!/bin/bash
# 2-GPU call: parity, fused-exchange timeline, N=2 bench with the fused exchanges on / off.
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29538 tests/dist_check.py > gpurun_out/dist_check_2f.log 2>&1; echo "dist_check 2 rc=$?"
grep -E '^\{' gpurun_out/dist_check_2f.log | grep -c '"ok": true'; grep -E '"ok": false' gpurun_out/dist_check_2f.log | cut -c1-400; grep -iE "error|trap" gpurun_out/dist_check_2f.log | head -5
BDDC_FUSED_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 tools/fused_trace.py > gpurun_out/fused_trace.log 2>&1; echo trace rc=$?
grep "^rank 0" gpurun_out/fused_trace.log
for F in 7 0 7 0; do
BDDC_FUSED_EX=$F timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2956$F bench.py --gpus 2 --steps 30 --warmup 3 > gpurun_out/f_n2_$F.log 2>&1; echo "bench 2 fused=$F rc=$?"; grep -iE "error" gpurun_out/f_n2_$F.log | head -3
python - $F <<'P'
import json,sys
W=sys.argv[1]
d=json.loads([l for l in open(f'gpurun_out/f_n2_{W}.log') if l.startswith('{')][-1])
print(W, round(d['ms_per_step'],3), round(d['value'],1), d['iterations'], round(d['apply']['ms'],4), round(d['roofline']['launch_ms'],4), round(d['e2e']['ms_per_step'],3), d['gpu_launches'])
P
done
