#!/bin/bash
mkdir -p gpurun_out/r02c
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_guards.py -q -rf --timeout 600 > gpurun_out/r02c/pytest_new.log 2>&1; echo "new rc $?"
timeout 900 python bench.py --steps 3 --warmup 3 --no-configs --no-cpu-baseline > gpurun_out/r02c/bench.log 2>&1; echo "bench rc $?"
