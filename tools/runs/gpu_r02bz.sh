#!/bin/bash
# K3 segment-factored exact terms (-DSE2_K3_SFMA build) against the committed kernel: timing + log-domain parity
OUT=gpurun_out/r02bz; mkdir -p $OUT
python tools/time_k3.py c1 c2 c3 2>&1 | cut -c1-200 | tee $OUT/head.log
SE2_LIB_PATH=$PWD/tools/k10/bin/libse2ot_sfma.so python tools/time_k3.py c1 c2 c3 2>&1 | cut -c1-200 | tee $OUT/sfma.log
SE2_LIB_PATH=$PWD/tools/k10/bin/libse2ot_sfma.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py -q -x --timeout 900 -k "log or lse or barycenter or sinkhorn or hint" > $OUT/pytest_sfma.log 2>&1; echo "rc $?"
tail -3 $OUT/pytest_sfma.log
