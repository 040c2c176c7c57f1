#!/bin/bash
OUT=gpurun_out/r02ao; mkdir -p $OUT
python tools/time_bary.py c3 > $OUT/timing.log 2>&1
