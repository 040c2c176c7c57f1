#!/bin/bash
# A/B the bench config sweep over library variants in variants/*.so (diagnostics only)
for so in variants/*.so; do
  echo "== $so"; SE2_LIB_PATH=$so python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k: (round(v['iters_per_s'],1), v.get('k3_exact_rows_live_frac'), v.get('k3_pairs',{}).get('hint_redos')) for k,v in d['configs'].items() if k in ('c1','c2','c3')})"
done
