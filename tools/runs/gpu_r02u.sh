#!/bin/bash
OUT=gpurun_out/r02u; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 1200 -k "c4w" > $OUT/pytest_c4w.log 2>&1; echo "c4w rc $?"
timeout 900 python -m pytest tests/test_gpu_lifting.py -q -rf --timeout 600 > $OUT/pytest_lift.log 2>&1; echo "lift rc $?"
