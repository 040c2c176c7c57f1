#!/bin/bash
# same-box A/B: the committed library (32 KB weight stages, ring of 4) against 64 KB stages, ring of 2
OUT=gpurun_out/r02bt; mkdir -p $OUT
for i in 1 2 3; do
python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/new.log 2>&1
SE2_LIB_PATH=$PWD/tools/k10/bin/libse2ot_head.so python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/head.log 2>&1
done
grep -H "ms/conv" $OUT/*.log | cut -c1-70
timeout 600 python -m pytest tests/test_gpu_ops.py -q -x --timeout 900 -k "tc" 2>&1 | tail -2
