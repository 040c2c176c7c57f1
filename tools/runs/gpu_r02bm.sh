#!/bin/bash
# ncu --set full of the K10 pieces epilogue and split kernels (c4, warm L2 as far as ncu allows)
OUT=gpurun_out/r02bm; mkdir -p $OUT
python tools/prof_conv.py --cfg c4 --reps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"tc_pieces_epilogue|tc_split_input" -s 2 -c 2 -o $OUT/k10_epi \
    python tools/prof_conv.py --cfg c4 --reps 2 > $OUT/ncu.log 2>&1
ncu -i $OUT/k10_epi.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ncu -i $OUT/k10_epi.ncu-rep --page source --csv > $OUT/src.csv 2>/dev/null
tail -3 $OUT/ncu.log
