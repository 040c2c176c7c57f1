#!/bin/bash
OUT=gpurun_out/r02v; mkdir -p $OUT
for c in 4 1 2 8 16; do echo "chain16 $c" >> $OUT/prof.log; SE2_TC_CHAIN16=$c python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prof.log 2>&1; done
