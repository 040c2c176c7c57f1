#!/bin/bash
# K10 diagnostics: no weight loads after the first ring fill, alone and with half-N MMAs
OUT=gpurun_out/r02bj; mkdir -p $OUT
for i in 1 2; do
SE2_TC_DIAG_SKIP_EPI=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_DIAG_NOWLOAD=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi_nowload.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_DIAG_HALFN=1 SE2_TC_DIAG_NOWLOAD=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi_halfn_nowload.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 SE2_TC_DIAG_HALFN=1 SE2_TC_CHAIN16=16 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/noepi_halfn_chain16.log 2>&1
done
grep -H "ms/conv" $OUT/*.log | cut -c1-120
