#!/bin/bash
OUT=gpurun_out/r02ah; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -rf --timeout 900 > $OUT/pytest_dist.log 2>&1; echo "dist rc $?"
