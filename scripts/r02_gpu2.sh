#!/bin/bash
# round-2 GPU call 2: two-team split kernel + Jacobi v2: parity (attention + factor), A/B bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_factor.py -m gpu -q --timeout 600 -x -p no:cacheprovider > gpurun_out/r02_pytest2.log 2>&1
echo PYTEST_RC=$? ; tail -15 gpurun_out/r02_pytest2.log
./scripts/fp64_rate > gpurun_out/r02_fp64_rate.log 2>&1; cat gpurun_out/r02_fp64_rate.log
timeout 300 python scripts/seal_cost.py --profile > gpurun_out/r02_seal2.json 2>&1; cat gpurun_out/r02_seal2.json | tail -1
for cfg in c2 c4 c3; do
timeout 600 bash scripts/lib_ab.sh $cfg "--config $cfg" base variants/teams1/libdquant_b200.so variants/pf2/libdquant_b200.so variants/pf5/libdquant_b200.so
done
