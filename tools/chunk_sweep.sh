for K in 8 16 32; do BDDC_MIN_CHUNK_ROWS=$K timeout 200 python tools/gpu_check.py c2 | python -c "
import ast,sys; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); kt=d['kernel_times']
print('min_kr', $K, 'apply_ms', round(d['apply_ms'],4), 'interior per launch', round(kt['interior_ms']/kt['interior_launches'],4), 'pcg_s', round(d['pcg_s'],5), d['iterations'], d['hist_rel_err'])"; done
