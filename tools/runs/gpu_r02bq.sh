#!/bin/bash
# K10: next stage's barrier poll between the current stage's MMA blocks, A/B + K10 tests
OUT=gpurun_out/r02bq; mkdir -p $OUT
for i in 1 2; do
python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/new.log 2>&1
SE2_TC_NO_PREPOLL=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/old.log 2>&1
done
SE2_TC_DIAG_PROF=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prof.log 2>&1
grep -H "ms/conv\|issuer" $OUT/*.log | cut -c1-170
timeout 1200 python -m pytest tests/test_gpu_ops.py -q -x --timeout 900 -k "tc" > $OUT/pytest_tc.log 2>&1; echo "tc rc $?"
tail -2 $OUT/pytest_tc.log
