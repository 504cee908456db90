#!/bin/bash
# round-2 GPU call 6: DMMA Gram / projection, NaN-safe sort; wait-hint A/B of the two-team kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_attention.py tests/test_gpu_kvcache.py tests/test_gpu_formats.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/r02_pytest6.log 2>&1
echo PYTEST_RC=$? ; tail -8 gpurun_out/r02_pytest6.log
timeout 300 python scripts/seal_cost.py --profile > gpurun_out/r02_seal6.json 2>&1; tail -1 gpurun_out/r02_seal6.json
timeout 900 bash scripts/lib_ab.sh p6 "--config c2" base variants/hint0/libdquant_b200.so variants/ns_t2/libdquant_b200.so variants/ns_t2h0/libdquant_b200.so variants/teams1/libdquant_b200.so
