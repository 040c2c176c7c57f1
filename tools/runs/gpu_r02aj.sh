#!/bin/bash
OUT=gpurun_out/r02aj; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_ops.py -q -rf --timeout 900 -k "precise" > $OUT/pytest_precise_ops.log 2>&1; echo "rc $?"
