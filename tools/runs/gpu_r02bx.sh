#!/bin/bash
# K10 chained convs: the pieces epilogue also writes the next conv's input split; A/B + tests
OUT=gpurun_out/r02bx; mkdir -p $OUT
for i in 1 2; do python tools/time_jko.py; SE2_TC_NO_CHAIN=1 python tools/time_jko.py; done 2>&1 | tee $OUT/time.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_ops.py tests/test_gpu_guards.py -q -x --timeout 900 -k "c4 or jko or tc or sinkhorn or linear or guard" > $OUT/pytest.log 2>&1; echo "rc $?"
tail -4 $OUT/pytest.log
