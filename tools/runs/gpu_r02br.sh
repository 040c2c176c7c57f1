#!/bin/bash
OUT=gpurun_out/r02br; mkdir -p $OUT
for i in 1 2 3; do
python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/new.log 2>&1
SE2_TC_NO_NEXTOPS=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prepoll_only.log 2>&1
SE2_TC_NO_PREPOLL=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/none.log 2>&1
done
grep -H "ms/conv" $OUT/*.log | cut -c1-70
