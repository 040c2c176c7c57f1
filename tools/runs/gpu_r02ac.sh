#!/bin/bash
OUT=gpurun_out/r02ac; mkdir -p $OUT
python tools/time_bary.py c1 c2 c3 > $OUT/timing.log 2>&1
for g in 1 3 5 8; do echo "groups $g" >> $OUT/timing_g.log; SE2_K4P_GROUPS=$g python tools/time_bary.py c1 c2 2>&1 | grep precise >> $OUT/timing_g.log; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py -q -rf --timeout 900 -k "precise and not c3m and not c3q" > $OUT/pytest_precise.log 2>&1; echo "precise rc $?"
