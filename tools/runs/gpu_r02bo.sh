#!/bin/bash
OUT=gpurun_out/r02bo; mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 60 --csv --log-file $OUT/l_new.csv python tools/prof_conv.py --cfg c4 --reps 8 > /dev/null 2>&1
SE2_TC_SPLIT1=1 SE2_TC_EPI1=1 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 60 --csv --log-file $OUT/l_old.csv python tools/prof_conv.py --cfg c4 --reps 8 > /dev/null 2>&1
python tools/k10/launch_times.py < $OUT/l_new.csv; python tools/k10/launch_times.py < $OUT/l_old.csv
