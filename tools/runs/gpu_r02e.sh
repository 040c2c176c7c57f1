#!/bin/bash
# r02 (re-entry) first GPU pass: smoke, the GPU suite (cases whose goldens are being regenerated
# deselected), the default bench line and the ncu launch list of a bench step.
OUT=gpurun_out/r02e; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?"
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 -k "not c3m and not c3q and not c4w and not c4f" \
    > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 900 python bench.py > $OUT/bench_default.log 2>&1; echo "bench rc $?"
timeout 600 python bench.py --steps 1 --warmup 1 --no-configs --no-cpu-baseline > $OUT/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $OUT/launches_c4.csv \
    python bench.py --steps 1 --warmup 1 --no-configs --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu rc $?"
