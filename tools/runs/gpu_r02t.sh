#!/bin/bash
OUT=gpurun_out/r02t; mkdir -p $OUT
(cd variants/old && python tools/time_bary.py c2 c3 > ../../$OUT/old.log 2>&1)
python tools/time_bary.py c2 c3 > $OUT/new.log 2>&1
