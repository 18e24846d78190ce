for L in 16 24 32 12; do LEAF=$L timeout 200 python tools/gpu_check.py c2 | python -c "
import ast,sys; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); kt=d['kernel_times']
print('leaf', $L, 'apply_ms', round(d['apply_ms'],4), 'interior per launch', round(kt['interior_ms']/kt['interior_launches'],4), 'factor', d['stats']['factor_values'], 'pcg_s', round(d['pcg_s'],5), d['iterations'], d['hist_rel_err'])"; done
