#!/bin/bash
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 1 > gpurun_out/bench_full.log 2>&1
for c in c2 c3; do for it in 10 100 300; do python tools/prof_state_conv.py --cfg $c --iters $it; done; done > gpurun_out/state_conv.log 2>&1
python tools/prof_state_conv.py --cfg c3 --iters 100 --exact >> gpurun_out/state_conv.log 2>&1
python bench.py --steps 1 --warmup 1 --no-configs --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_c4_r01.csv \
    python bench.py --steps 1 --warmup 1 --no-configs --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/prof_conv.py --cfg c4 --reps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_linear -s 1 -c 1 -o gpurun_out/prof_c4_linear_v2 \
    python tools/prof_conv.py --cfg c4 --reps 2 > gpurun_out/ncu_full_c4.log 2>&1
python tools/prof_state_conv.py --cfg c3 --iters 100 --reps 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_lse_fast -s 1 -c 1 -o gpurun_out/prof_c3_k3 \
    python tools/prof_state_conv.py --cfg c3 --iters 100 --reps 1 > gpurun_out/ncu_full_c3.log 2>&1
echo done
