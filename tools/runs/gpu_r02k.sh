#!/bin/bash
OUT=gpurun_out/r02k; mkdir -p $OUT
for na in 6 8 4; do echo "na $na" >> $OUT/prof.log; SE2_TC_NA=$na python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prof.log 2>&1; done
echo "rows mode" >> $OUT/prof.log; SE2_TC_PIECES=0 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prof.log 2>&1
echo "classic" >> $OUT/prof.log; SE2_TC_NAR=0 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prof.log 2>&1
echo "classic rows" >> $OUT/prof.log; SE2_TC_PIECES=0 SE2_TC_NAR=0 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prof.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> $OUT/prof.log
timeout 1200 python -m pytest tests/test_gpu_ops.py -q -rf --timeout 600 -k "tc or narrow" > $OUT/pytest_tc.log 2>&1; echo "tc rc $?"
