#!/bin/bash
# K10 with elect.sync roles (no per-instruction ELECT loops): timing + the K10 tests
OUT=gpurun_out/r02bh; mkdir -p $OUT
for i in 1 2; do
python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/base.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_DIAG_HALFN=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi_halfn.log 2>&1
done
grep -H "ms/conv" $OUT/*.log | cut -c1-120
timeout 1200 python -m pytest tests/test_gpu_ops.py tests/test_gpu_parity.py -q -x --timeout 900 -k "tc or c4 or linear" > $OUT/pytest_tc.log 2>&1; echo "tc rc $?"
tail -3 $OUT/pytest_tc.log
