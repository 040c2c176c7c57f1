#!/bin/bash
# full validation + measurement pass after the K10 narrow geometry
OUT=gpurun_out/r02o; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?"
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 -k "not c3m and not c3q and not c4w and not c4f" \
    > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 900 python bench.py > $OUT/bench_default.log 2>&1; echo "bench rc $?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.log 2>&1; echo "ref rc $?"
timeout 600 python bench.py --steps 1 --warmup 1 --no-configs --no-cpu-baseline > $OUT/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $OUT/launches_c4.csv \
    python bench.py --steps 1 --warmup 1 --no-configs --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu launch rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_tc_kernel|tc_split_input|tc_pieces_epilogue" -s 3 -c 3 -o $OUT/k10_c4 \
    python tools/prof_conv.py --cfg c4 --reps 2 > $OUT/ncu_full.log 2>&1; echo "ncu full rc $?"
