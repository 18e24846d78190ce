#!/bin/bash
# compute-sanitizer is closed on this pool: run the single-GPU test suite against the checked
# build (every interior-solve tile access bounds-checked, a violation traps), then restore
mkdir -p gpurun_out
cp paper_2410_14786_b200/lib/libbddc_b200.so /tmp/libdefault.so
cp paper_2410_14786_b200/lib/libbddc_b200_checked.so paper_2410_14786_b200/lib/libbddc_b200.so
timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_distributed.py > gpurun_out/pytest_checked.log 2>&1; echo "checked pytest rc $?"
tail -3 gpurun_out/pytest_checked.log
timeout 600 python bench.py --no-cpu-baseline --no-extra --steps 5 > gpurun_out/bench_checked.jsonl 2> gpurun_out/bench_checked.err; echo "checked bench rc $?"
cp /tmp/libdefault.so paper_2410_14786_b200/lib/libbddc_b200.so
