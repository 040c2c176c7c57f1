#!/bin/bash
OUT=gpurun_out/r02j; mkdir -p $OUT
for e in 0 1 2 3 4; do echo "early $e" >> $OUT/prof.log; SE2_TC_EARLY=$e python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prof.log 2>&1; done
SE2_TC_NAR=0 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prof.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_ops.py -q -rf --timeout 600 -k "tc or narrow" > $OUT/pytest_tc.log 2>&1; echo "tc rc $?"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 900 -k "jko and (c4q or c4p or c4m or c5m)" > $OUT/pytest_jko.log 2>&1; echo "jko rc $?"
