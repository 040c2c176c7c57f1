#!/bin/bash
OUT=gpurun_out/r02ag; mkdir -p $OUT
python tools/time_bary.py c1 c2 c3 > $OUT/timing.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py -q -rf --timeout 900 -k "(log or lse or barycenter or sinkhorn or hint) and not c3q" > $OUT/pytest_log.log 2>&1; echo "log rc $?"
python tools/run_bary.py --cfg c3 --iters 210 --no-graph > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_lse_fast -s 400 -c 1 -o $OUT/k3_c3 python tools/run_bary.py --cfg c3 --iters 210 --no-graph > $OUT/ncu.log 2>&1
