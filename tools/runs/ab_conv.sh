#!/bin/bash
# A/B the c4 linear conv over library variants in variants/*.so (diagnostics only)
for so in variants/*.so; do echo "== $so"; SE2_LIB_PATH=$so python tools/prof_conv.py --cfg c4 --reps 20; done
