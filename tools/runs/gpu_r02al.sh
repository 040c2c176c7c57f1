#!/bin/bash
OUT=gpurun_out/r02al; mkdir -p $OUT
python tools/prof_conv.py --cfg c4 --reps 50 > $OUT/prof.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 python tools/prof_conv.py --cfg c4 --reps 50 >> $OUT/prof.log 2>&1
SE2_TC_DIAG_SKIP_SPLIT=1 python tools/prof_conv.py --cfg c4 --reps 50 >> $OUT/prof.log 2>&1
SE2_TC_DIAG_SKIP_SPLIT=1 SE2_TC_DIAG_SKIP_EPI=1 python tools/prof_conv.py --cfg c4 --reps 50 >> $OUT/prof.log 2>&1
