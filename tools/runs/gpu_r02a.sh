#!/bin/bash
# r02 first GPU pass: parity suite under the restored elementwise metric + compute-sanitizer
mkdir -p gpurun_out/r02a
cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02a/smoke.log 2>&1; echo "smoke rc $?"
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 -k "not c3m and not c3q and not c4w and not c4f" \
    > gpurun_out/r02a/pytest_gpu.log 2>&1; echo "pytest rc $?"
SAN=/usr/local/cuda/bin/compute-sanitizer
for spec in "racecheck k10" "racecheck k9 k3 slab bary" "synccheck k10 k9 k3 slab bary" "memcheck all" "initcheck k10 k2 k9"; do
    set -- $spec; tool=$1; shift
    timeout 900 $SAN --tool $tool --print-limit 50 python tools/sanitize.py "$@" > gpurun_out/r02a/san_${tool}_$(echo "$@" | tr ' ' '_').log 2>&1
    echo "$tool $@ rc $?"
done
