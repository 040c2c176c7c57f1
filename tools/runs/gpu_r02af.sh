#!/bin/bash
OUT=gpurun_out/r02af; mkdir -p $OUT
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 1500 -k "c3m" > $OUT/pytest_c3m.log 2>&1; echo "c3m rc $?"
