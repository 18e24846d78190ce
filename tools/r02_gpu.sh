#!/bin/bash
# round-2 GPU check: pytest -m gpu, then the default bench line (C2 + extra configs + cpu baselines)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc $?"
tail -c 3000 gpurun_out/bench.jsonl
