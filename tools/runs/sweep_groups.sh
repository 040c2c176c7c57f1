#!/bin/bash
for g in 1 2 3 4 5 6 7 8; do
  echo "groups $g"; SE2_K3_GROUPS=$g python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v['iters_per_s'],1) for k,v in d['configs'].items() if k in ('c1','c2','c3')})"
done
