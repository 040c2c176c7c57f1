#!/bin/bash
# full GPU validation + measurement pass (one gpurun call)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/pytest_gpu_all.log 2>&1
python bench.py > gpurun_out/bench_default.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1
python bench.py --steps 1 --warmup 1 --no-configs --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --steps 1 --warmup 1 --no-configs --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/prof_conv.py --cfg c4 --reps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 1 -c 1 -o gpurun_out/prof_c4_tc \
    python tools/prof_conv.py --cfg c4 --reps 2 > gpurun_out/ncu_full_c4_tc.log 2>&1
SE2_NO_TC=1 python tools/prof_conv.py --cfg c4 --reps 2 > /dev/null 2>&1 && \
SE2_NO_TC=1 ncu --set full --clock-control none --import-source on -k regex:conv_linear -s 1 -c 1 -o gpurun_out/prof_c4_linear \
    python tools/prof_conv.py --cfg c4 --reps 2 > gpurun_out/ncu_full_c4.log 2>&1
python tools/run_bary.py --cfg c3 --iters 210 --no-graph > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_lse_fast -s 400 -c 1 -o gpurun_out/prof_c3_k3_solve \
    python tools/run_bary.py --cfg c3 --iters 210 --no-graph > gpurun_out/ncu_full_c3.log 2>&1
python tools/run_sinkhorn.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sinkhorn_small -s 1 -c 1 -o gpurun_out/prof_c0_k9 \
    python tools/run_sinkhorn.py > gpurun_out/ncu_full_c0.log 2>&1
echo done
