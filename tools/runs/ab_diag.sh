#!/bin/bash
# A/B the parity diagnostics over library variants in variants/*.so (diagnostics only)
for so in variants/*.so; do
  for c in c2m c3m c1; do
    echo "== $so $c"; SE2_LIB_PATH=$so python tools/diag_c1.py $c 2>&1 | grep -E "measure err floor 1e-06|lbary err" | head -12
  done
done
