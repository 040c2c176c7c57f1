#!/bin/bash
# NCCL transport on one GPU (one-rank communicator), the dist suite, the bench contract with the manifest
OUT=gpurun_out/r02bl; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_contract.py tests/test_gpu_parallel.py -q -x --timeout 900 > $OUT/pytest.log 2>&1; echo "rc $?"
tail -15 $OUT/pytest.log
