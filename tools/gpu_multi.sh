#!/bin/bash
# multi-GPU evidence (run with gpurun --gpus 4): distributed parity incl. C3 and the N=8 layout on
# 4 GPUs, weak-scaling bench lines N=2/4, the 32x16 layout bench at N=4, fused-exchange trace
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l); echo "gpus $N"
timeout 2400 python -m pytest tests/test_gpu_distributed.py -q -s > gpurun_out/pytest_dist.log 2>&1; echo "dist rc $?"
grep -E '^\{"config"' gpurun_out/pytest_dist.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['rank']==0: print(d['world'], d['config'], d['ok'], d['apply_bitwise'], d['iterations'], '%.2e'%d.get('history_err_vs_reference',-1))
"
tail -3 gpurun_out/pytest_dist.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/bench_n$n.jsonl 2> gpurun_out/bench_n$n.err; echo "bench n$n rc $?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --steps 20 --warmup 3 --subdomains 32x16 --no-extra > gpurun_out/bench_n4_32x16.jsonl 2> gpurun_out/bench_n4_32x16.err; echo "bench 32x16 rc $?"
LAYOUT=32x16 BDDC_FUSED_TRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 tools/fused_trace.py > gpurun_out/fused_trace_32x16.txt 2>&1; echo "trace rc $?"
tail -20 gpurun_out/fused_trace_32x16.txt
for f in gpurun_out/bench_n2.jsonl gpurun_out/bench_n4.jsonl gpurun_out/bench_n4_32x16.jsonl; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'setup', round(d['setup_seconds'],3), {k:(round(e['ms_per_step'],3), e['iterations']) for k,e in (d.get('extra_configs') or {}).items()})"; done
