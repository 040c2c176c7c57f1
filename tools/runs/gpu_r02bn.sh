#!/bin/bash
# K10: 4-pixel split kernel and 4-output pieces epilogue, A/B against the scalar forms + the K10 / c4 tests
OUT=gpurun_out/r02bn; mkdir -p $OUT
for i in 1 2; do
python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/new.log 2>&1
SE2_TC_SPLIT1=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/split1.log 2>&1
SE2_TC_EPI1=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/epi1.log 2>&1
SE2_TC_SPLIT1=1 SE2_TC_EPI1=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/old.log 2>&1
done
grep -H "ms/conv" $OUT/*.log | cut -c1-110
timeout 1500 python -m pytest tests/test_gpu_ops.py tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_guards.py -q -x --timeout 900 -k "tc or c4 or linear or jko or guard" > $OUT/pytest_tc.log 2>&1; echo "tc rc $?"
tail -3 $OUT/pytest_tc.log
python bench.py --steps 3 --warmup 3 --no-configs --no-cpu-baseline > $OUT/bench.log 2>&1; cut -c1-400 $OUT/bench.log
