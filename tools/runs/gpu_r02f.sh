#!/bin/bash
# K10 narrow geometry: parity of the tensor-core conv + JKO, then a bench step
OUT=gpurun_out/r02f; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?"
timeout 1200 python -m pytest tests/test_gpu_ops.py -q -rf --timeout 600 -k "tc or narrow" > $OUT/pytest_tc.log 2>&1; echo "tc rc $?"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 900 -k "jko and (c4q or c4p or c4m)" > $OUT/pytest_jko.log 2>&1; echo "jko rc $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-configs --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc $?"
SE2_TC_NAR=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-configs --no-cpu-baseline > $OUT/bench_classic.log 2>&1; echo "bench classic rc $?"
