#!/bin/bash
OUT=gpurun_out/r02p; mkdir -p $OUT
python tools/conv_err_probe.py c1 > $OUT/probe_c1.log 2>&1
python tools/conv_err_probe.py c2m > $OUT/probe_c2m.log 2>&1
