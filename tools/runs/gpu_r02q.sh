#!/bin/bash
# compute-sanitizer evidence (SURVEY.md:282): racecheck / synccheck / memcheck / initcheck on the hot kernels
OUT=gpurun_out/r02q; mkdir -p $OUT
SAN=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize.py all > $OUT/plain.log 2>&1; echo "plain rc $?"
for spec in "racecheck k10" "racecheck k9 k3 slab bary precise" "synccheck k10 k9 k3 slab bary precise" "memcheck all" "initcheck k10 k2 k9 precise"; do
    set -- $spec; tool=$1; shift
    timeout 900 $SAN --tool $tool --print-limit 50 python tools/sanitize.py "$@" > $OUT/san_${tool}_$(echo "$@" | tr ' ' '_').log 2>&1
    echo "$tool $@ rc $?"
done
