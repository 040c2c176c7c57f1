#!/bin/bash
# K10: griddepcontrol.launch_dependents at the top of the three kernels, A/B + tests
OUT=gpurun_out/r02bw; mkdir -p $OUT
for i in 1 2 3; do
python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/new.log 2>&1
SE2_TC_NO_PDL_EARLY=1 python tools/prof_conv.py --cfg c4 --reps 20 >> $OUT/old.log 2>&1
done
grep -H "ms/conv" $OUT/*.log | cut -c1-70
python tools/time_slab_conv.py 8 | tail -1; SE2_TC_NO_PDL_EARLY=1 python tools/time_slab_conv.py 8 | tail -1
timeout 1200 python -m pytest tests/test_gpu_ops.py tests/test_gpu_parity.py -q -x --timeout 900 -k "tc or c4" 2>&1 | tail -2
