#!/bin/bash
# K10 fine balance on thin output windows: slab conv timings (1 / 2 / 4 / 8 slabs), the K10 / dist tests
OUT=gpurun_out/r02bu; mkdir -p $OUT
python tools/time_slab_conv.py > $OUT/slab_new.log 2>&1; cat $OUT/slab_new.log
timeout 1500 python -m pytest tests/test_gpu_ops.py tests/test_gpu_dist.py tests/test_gpu_parallel.py -q -x --timeout 900 -k "tc or jko or slab or window" > $OUT/pytest.log 2>&1; echo "rc $?"
tail -3 $OUT/pytest.log
