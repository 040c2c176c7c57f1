#!/bin/bash
# K10: does the weight stream cost MMA time?  (SE2_TC_DIAG_HALFW halves the weight bytes per stage; results wrong)
OUT=gpurun_out/r02bd; mkdir -p $OUT
for i in 1 2; do
python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/base.log 2>&1
SE2_TC_DIAG_HALFW=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/halfw.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_DIAG_SKIP_SPLIT=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/mma_only.log 2>&1
SE2_TC_DIAG_HALFW=1 SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_DIAG_SKIP_SPLIT=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/mma_only_halfw.log 2>&1
done
grep -H "ms/conv" $OUT/*.log | cut -c1-120
