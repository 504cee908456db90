#!/bin/bash
# prepare kernels on FFMA2, combine merges with their loads batched: parity, then A/B on C5 / C2 / C4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_asym.py tests/test_gpu_sharding.py -q -x -m gpu > gpurun_out/r02_g55_tests.log 2>&1; echo TESTS=$?
tail -2 gpurun_out/r02_g55_tests.log
timeout 400 bash scripts/lib_ab.sh g55c5 "--config c5 --layers 16" base variants/gq_old/libdquant_b200.so
timeout 300 bash scripts/lib_ab.sh g55c2 "" base variants/gq_old/libdquant_b200.so
timeout 300 bash scripts/lib_ab.sh g55c4 "--config c4" base variants/gq_old/libdquant_b200.so
