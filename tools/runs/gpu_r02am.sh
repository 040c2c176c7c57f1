#!/bin/bash
OUT=gpurun_out/r02am; mkdir -p $OUT
python tools/prof_conv.py --cfg c4 --reps 50 > $OUT/prof.log 2>&1
SE2_TC_DIAG_SKIP_EPI=1 python tools/prof_conv.py --cfg c4 --reps 50 >> $OUT/prof.log 2>&1
python tools/prof_conv.py --cfg c4 --reps 50 >> $OUT/prof.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-configs --no-cpu-baseline > $OUT/bench.log 2>&1
