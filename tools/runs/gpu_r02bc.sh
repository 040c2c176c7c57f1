#!/bin/bash
# r02 re-entry check of HEAD: smoke, the whole GPU suite, the default bench line
OUT=gpurun_out/r02bc; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?"
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -4 $OUT/pytest_gpu.log
python bench.py > $OUT/bench.log 2> $OUT/bench.err; echo "bench rc $?"
tail -c 600 $OUT/bench.log
