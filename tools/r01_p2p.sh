#!/bin/bash
# 2-GPU call: distributed parity with peer-memory exchanges, bench N=2 (P2P vs NCCL).
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tests/dist_check.py > gpurun_out/dist_check_p2p.log 2>&1; echo "dist_check rc=$?"
grep -E '^\{' gpurun_out/dist_check_p2p.log | grep -c '"ok": true'; grep -E '"ok": false' gpurun_out/dist_check_p2p.log | cut -c1-500; grep -iE "error" gpurun_out/dist_check_p2p.log | head -5
for P in 1 0; do
BDDC_P2P=$P timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954$P bench.py --gpus 2 --steps 30 --warmup 3 > gpurun_out/bench_n2_p2p$P.log 2>&1; echo "bench p2p=$P rc=$?"; grep -iE "error" gpurun_out/bench_n2_p2p$P.log | head -3
python - $P <<'X'
import json,sys
d=json.loads([l for l in open(f'gpurun_out/bench_n2_p2p{sys.argv[1]}.log') if l.startswith('{')][-1])
print(round(d['ms_per_step'],3), round(d['value'],1), d['iterations'], round(d['apply']['ms'],4), round(d['e2e']['ms_per_step'],3))
X
done
