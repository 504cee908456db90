#!/bin/bash
# round-2 GPU call 3: producer rewrite + K3 fast path: parity, seal cost, A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_factor.py tests/test_gpu_codec.py tests/test_gpu_kvcache.py -m gpu -q --timeout 600 -x -p no:cacheprovider > gpurun_out/r02_pytest3.log 2>&1
echo PYTEST_RC=$? ; tail -5 gpurun_out/r02_pytest3.log
DQ_LIB=variants/jstats/libdquant_b200.so timeout 300 python scripts/seal_cost.py --units 4 2>&1 | grep jacobi | head -4
DQ_LIB=variants/jstats16/libdquant_b200.so timeout 300 python scripts/seal_cost.py --units 4 2>&1 | grep jacobi | head -4
timeout 300 python scripts/seal_cost.py --profile > gpurun_out/r02_seal3.json 2>&1; tail -1 gpurun_out/r02_seal3.json
for cfg in c2 c4 c3; do
timeout 600 bash scripts/lib_ab.sh $cfg "--config $cfg" base variants/teams1/libdquant_b200.so variants/pf5/libdquant_b200.so
done
