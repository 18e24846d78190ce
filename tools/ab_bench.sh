# A/B of environment variants on the C2 bench line, interleaved rounds (VARIANTS, ROUNDS)
mkdir -p gpurun_out
for rnd in $(seq 1 ${ROUNDS:-3}); do
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then envs=""; else envs="${v//+/ }"; fi
  env $envs timeout 600 python bench.py --no-cpu-baseline --no-extra --steps ${STEPS:-30} ${BENCH_ARGS} > gpurun_out/ab.jsonl 2>gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.jsonl').read().strip().splitlines()[-1])
print('$rnd $v ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'launch', round(d['roofline']['launch_ms'],4), 'apply', round(d['apply']['ms'],4), 'it', d['iterations'], 'clk', d['clocks']['sm_mhz'])
" || tail -5 gpurun_out/ab.err
done; done
