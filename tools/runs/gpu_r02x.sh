#!/bin/bash
OUT=gpurun_out/r02x; mkdir -p $OUT
python tools/time_bary.py c1 c2 c3 > $OUT/timing.log 2>&1; echo "timing rc $?"
SE2_K4P_EXACT=1 python tools/time_bary.py c2 > $OUT/timing_exact.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py -q -rf --timeout 900 -k "precise and not c3m and not c3q" > $OUT/pytest_precise.log 2>&1; echo "precise rc $?"
