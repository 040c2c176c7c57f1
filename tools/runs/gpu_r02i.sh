#!/bin/bash
OUT=gpurun_out/r02i; mkdir -p $OUT
python tools/prof_conv.py --cfg c4 --reps 20 > $OUT/prof.log 2>&1; echo "prof rc $?"
SE2_TC_NAR=0 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/prof.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_ops.py -q -rf --timeout 600 -k "tc or narrow" > $OUT/pytest_tc.log 2>&1; echo "tc rc $?"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 900 -k "jko and (c4q or c4p or c4m or c5m)" > $OUT/pytest_jko.log 2>&1; echo "jko rc $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-configs --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 1 -c 1 -o $OUT/nar_c4 \
    python tools/prof_conv.py --cfg c4 --reps 2 > $OUT/ncu.log 2>&1
