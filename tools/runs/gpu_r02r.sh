#!/bin/bash
OUT=gpurun_out/r02r; mkdir -p $OUT
python tools/prof_conv.py --cfg c4 --reps 20 > $OUT/prof.log 2>&1; echo "prof rc $?"
timeout 1200 python -m pytest tests/test_gpu_ops.py -q -rf --timeout 600 -k "tc or narrow" > $OUT/pytest_tc.log 2>&1; echo "tc rc $?"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 900 -k "jko and (c4q or c4p or c4m or c5m)" > $OUT/pytest_jko.log 2>&1; echo "jko rc $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-configs --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc $?"
timeout 900 ncu --set full --clock-control none -k regex:"tc_pieces_epilogue" -s 3 -c 1 -o $OUT/epi_c4 python tools/prof_conv.py --cfg c4 --reps 2 > $OUT/ncu.log 2>&1
