#!/bin/bash
# K3 theta_i-split sweep on the small/mid configs (bench config sweep only)
for m in 592 1184 2368 4736; do
  echo "split_min $m"; SE2_K3_SPLIT_MIN=$m python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v['iters_per_s'],1) for k,v in d['configs'].items() if k in ('c1','c2','c3')})"
done
