#!/bin/bash
# K10 diagnostics combined: half-N MMAs with half the weight bytes (is the half-N time the L2 weight stream?)
OUT=gpurun_out/r02bi; mkdir -p $OUT
for i in 1 2; do
SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_DIAG_HALFN=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi_halfn.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_DIAG_HALFN=1 SE2_TC_DIAG_HALFW=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi_halfn_halfw.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_DIAG_HALFW=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi_halfw.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_NA=6 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi_na6.log 2>&1
done
grep -H "ms/conv" $OUT/*.log | cut -c1-120
