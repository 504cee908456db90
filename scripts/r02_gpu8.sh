#!/bin/bash
# round-2 GPU call 7: fetcher warp + batched producer rounds
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -m gpu -q --timeout 600 -x -p no:cacheprovider > gpurun_out/r02_pytest8.log 2>&1
echo PYTEST_RC=$? ; tail -4 gpurun_out/r02_pytest8.log
timeout 900 bash scripts/lib_ab.sh p8 "--config c2" base variants/ns_t2/libdquant_b200.so variants/teams1/libdquant_b200.so variants/ns_t1/libdquant_b200.so variants/pf5/libdquant_b200.so variants/pf8/libdquant_b200.so
