#!/bin/bash
OUT=gpurun_out/r02ab; mkdir -p $OUT
python tools/time_bary.py c1 c2 c3 > $OUT/timing.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py -q -rf --timeout 900 -k "precise and not c3m and not c3q" > $OUT/pytest_precise.log 2>&1; echo "precise rc $?"
ncu --set full --clock-control none --import-source on -k regex:conv_lse_precise -s 400 -c 1 -o $OUT/k4p_c3 python tools/run_bary_precise.py c3 220 > $OUT/ncu3.log 2>&1
