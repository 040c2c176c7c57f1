#!/bin/bash
OUT=gpurun_out/r02ad; mkdir -p $OUT
ncu --set full --clock-control none --import-source on -k regex:conv_lse_precise -s 400 -c 1 -o $OUT/k4p_c3 python tools/run_bary_precise.py c3 220 > $OUT/ncu3.log 2>&1
