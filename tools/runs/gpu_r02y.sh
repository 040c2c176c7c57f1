#!/bin/bash
OUT=gpurun_out/r02y; mkdir -p $OUT
for A in 0 2 4 6 8 100; do echo "A=$A" >> $OUT/timing.log; SE2_K4P_FFMA_A=$A python tools/time_bary.py c1 c2 c3 2>&1 | grep precise >> $OUT/timing.log; done
