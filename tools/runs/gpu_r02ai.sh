#!/bin/bash
OUT=gpurun_out/r02ai; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?"
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 1200 -k "not c3q and not c4f" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 1500 python bench.py > $OUT/bench_default.log 2>&1; echo "bench rc $?"
