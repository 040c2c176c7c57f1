#!/bin/bash
# one gpurun call: launch list of the bench step + ncu --set full of the conv kernels
set -x
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
for c in c4 c3; do python tools/prof_conv.py --cfg $c --reps 3 >> gpurun_out/prof_plain.log 2>&1; done
python tools/prof_conv.py --cfg c3 --log --reps 2 >> gpurun_out/prof_plain.log 2>&1
python tools/prof_conv.py --cfg c2 --log --batch 2 --reps 2 >> gpurun_out/prof_plain.log 2>&1
python tools/prof_conv.py --cfg c4 --reps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_linear -s 1 -c 1 -o gpurun_out/prof_c4_linear \
    python tools/prof_conv.py --cfg c4 --reps 2 > gpurun_out/ncu_full_c4.log 2>&1
python tools/prof_conv.py --cfg c3 --log --reps 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_lse -s 1 -c 1 -o gpurun_out/prof_c3_lse \
    python tools/prof_conv.py --cfg c3 --log --reps 1 > gpurun_out/ncu_full_c3.log 2>&1
echo done
