#!/bin/bash
mkdir -p gpurun_out/r02b
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_guards.py -q -rf --timeout 600 > gpurun_out/r02b/pytest_new.log 2>&1; echo "new rc $?"
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 -k "not c3m and not c3q and not c4w and not c4f and not test_gpu_dist and not test_gpu_guards" \
    > gpurun_out/r02b/pytest_gpu.log 2>&1; echo "pytest rc $?"
