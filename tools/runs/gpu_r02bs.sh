#!/bin/bash
# same-box A/B: the committed library (HEAD) against the working tree (pre-polls + next-stage operands)
OUT=gpurun_out/r02bs; mkdir -p $OUT
for i in 1 2 3; do
python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/new.log 2>&1
SE2_LIB_PATH=$PWD/tools/k10/bin/libse2ot_head.so python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/head.log 2>&1
SE2_TC_NO_NEXTOPS=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prepoll_only.log 2>&1
done
grep -H "ms/conv" $OUT/*.log | cut -c1-70
