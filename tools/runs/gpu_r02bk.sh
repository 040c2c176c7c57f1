#!/bin/bash
# K10 issuer cycle profile (SE2_TC_DIAG_PROF), full-N and half-N
OUT=gpurun_out/r02bk; mkdir -p $OUT
SE2_TC_DIAG_PROF=1 python tools/prof_conv.py --cfg c4 --reps 20 > $OUT/prof.log 2>&1
SE2_TC_DIAG_PROF=1 SE2_TC_DIAG_HALFN=1 python tools/prof_conv.py --cfg c4 --reps 20 > $OUT/prof_halfn.log 2>&1
SE2_TC_DIAG_PROF=1 SE2_TC_DIAG_HALFN=1 SE2_TC_DIAG_NOWLOAD=1 python tools/prof_conv.py --cfg c4 --reps 20 > $OUT/prof_halfn_nowload.log 2>&1
tail -3 $OUT/*.log | cut -c1-200
