#!/bin/bash
# K10: do pixel-shifted (not 128-byte aligned) B descriptors slow the MMAs?  (SE2_TC_DIAG_NOSHIFT: every filter
# column reads the aligned row start; results wrong)
OUT=gpurun_out/r02be; mkdir -p $OUT
for i in 1 2; do
python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/base.log 2>&1
SE2_TC_DIAG_NOSHIFT=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noshift.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_DIAG_NOSHIFT=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi_noshift.log 2>&1
done
grep -H "ms/conv" $OUT/*.log | cut -c1-120
