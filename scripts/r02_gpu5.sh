#!/bin/bash
# round-2 GPU call 5: converged producer warp, tridiagonal eigensolver
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_attention.py -m gpu -q --timeout 600 -x -p no:cacheprovider > gpurun_out/r02_pytest5.log 2>&1
echo PYTEST_RC=$? ; tail -5 gpurun_out/r02_pytest5.log
timeout 300 python scripts/seal_cost.py --profile > gpurun_out/r02_seal5.json 2>&1; tail -1 gpurun_out/r02_seal5.json
timeout 900 bash scripts/lib_ab.sh p5 "--config c2" base variants/teams1/libdquant_b200.so variants/ns_t2/libdquant_b200.so variants/ns_t1/libdquant_b200.so
