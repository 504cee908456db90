#!/bin/bash
# cross-item GQA schedule: parity (gqa tests) then C5 A/B against the previous schedule and KA variants
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -m gpu -k "gqa or c5 or g8 or kernel_g" > gpurun_out/r02_g20_tests.log 2>&1; echo TESTS=$?
tail -3 gpurun_out/r02_g20_tests.log
for L in variants/ka2/libdquant_b200.so; do
  DQ_LIB=$L timeout 300 python -m pytest tests/test_gpu_attention.py -q -x -m gpu -k "gqa or c5" > gpurun_out/r02_g20_tests_ka2.log 2>&1; echo TESTS_KA2=$?
done
timeout 900 bash scripts/lib_ab.sh g20 "--config c5" base variants/gq_old/libdquant_b200.so variants/ka2/libdquant_b200.so variants/ka4/libdquant_b200.so
