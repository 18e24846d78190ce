# timing experiments for the interior solve (dev tool)
for a in 1 3 12; do
  echo "l2_ahead=$a"; BDDC_L2_AHEAD=$a timeout 60 python tools/gpu_check.py c2 2>&1 | grep -o "'kernel_times': {[^}]*}"
done
