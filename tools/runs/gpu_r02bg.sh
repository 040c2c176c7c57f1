#!/bin/bash
# K10: tensor-bound or issue-bound?  SE2_TC_DIAG_HALFN issues the same MMA sequence at half the N (64 cycles each; results wrong)
OUT=gpurun_out/r02bg; mkdir -p $OUT
for i in 1 2; do
SE2_TC_DIAG_SKIP_EPI=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_DIAG_HALFN=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi_halfn.log 2>&1
done
grep -H "ms/conv" $OUT/*.log | cut -c1-120
