#!/bin/bash
OUT=gpurun_out/r02g; mkdir -p $OUT
python tools/prof_conv.py --cfg c4 --reps 20 > $OUT/prof.log 2>&1
SE2_TC_NAR=0 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prof.log 2>&1
SE2_TC_PIECES=0 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 1 -c 1 -o $OUT/nar_c4 \
    python tools/prof_conv.py --cfg c4 --reps 2 > $OUT/ncu.log 2>&1
echo done
