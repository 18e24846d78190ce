# timing experiments for the interior solve (dev tool)
for j in 0.5 1 2 4; do
  echo "jpw=$j"; BDDC_JOBS_PER_WARP=$j timeout 60 python tools/gpu_check.py c2 2>&1 | grep -o "'kernel_times': {[^}]*}\|'hist_rel_err': [0-9.e-]*"
done
