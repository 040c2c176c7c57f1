#!/bin/bash
# K10 issuer cycle profile with the loads / flushes removed one by one
OUT=gpurun_out/r02bp; mkdir -p $OUT
run() { echo "== $1" >> $OUT/prof.log; env $1 SE2_TC_DIAG_PROF=1 SE2_TC_DIAG_SKIP_EPI=1 python tools/prof_conv.py --cfg c4 --reps 20 2>&1 | cut -c1-160 >> $OUT/prof.log; }
run "X=1"
run "SE2_TC_DIAG_NOWLOAD=1"
run "SE2_TC_DIAG_NOBLOAD=1"
run "SE2_TC_DIAG_NOWLOAD=1 SE2_TC_DIAG_NOBLOAD=1"
run "SE2_TC_DIAG_NOWLOAD=1 SE2_TC_DIAG_NOBLOAD=1 SE2_TC_CHAIN16=16"
cat $OUT/prof.log
