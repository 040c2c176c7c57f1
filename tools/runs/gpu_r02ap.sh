#!/bin/bash
OUT=gpurun_out/r02ap; mkdir -p $OUT
python tools/prof_conv.py --cfg c4 --reps 50 > $OUT/prof.log 2>&1; echo "prof rc $?"
timeout 1200 python -m pytest tests/test_gpu_ops.py -q -rf --timeout 600 -k "tc or narrow or transport" > $OUT/pytest_tc.log 2>&1; echo "tc rc $?"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -rf --timeout 900 -k "jko" > $OUT/pytest_jko.log 2>&1; echo "jko rc $?"
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py --steps 5 --warmup 3 --no-configs --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc $?"
