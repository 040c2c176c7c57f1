#!/bin/bash
OUT=gpurun_out/r02z; mkdir -p $OUT
for A in 0 100; do echo "A=$A" >> $OUT/timing.log; SE2_K4P_FFMA_A=$A python tools/time_bary.py c1 c2 c3 2>&1 | grep precise >> $OUT/timing.log; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py -q -rf --timeout 900 -k "precise and not c3m and not c3q" > $OUT/pytest_precise.log 2>&1; echo "precise rc $?"
