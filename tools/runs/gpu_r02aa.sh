#!/bin/bash
OUT=gpurun_out/r02aa; mkdir -p $OUT
python tools/run_bary_precise.py c2 30 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c2p.csv python tools/run_bary_precise.py c2 30 > $OUT/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_lse_precise -s 60 -c 1 -o $OUT/k4p_c2 python tools/run_bary_precise.py c2 40 > $OUT/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_lse_precise -s 400 -c 1 -o $OUT/k4p_c3 python tools/run_bary_precise.py c3 220 > $OUT/ncu3.log 2>&1
echo done
