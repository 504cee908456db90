#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -m gpu -q --timeout 600 -x -p no:cacheprovider > gpurun_out/r02_pytest11.log 2>&1
echo PYTEST_RC=$? ; tail -3 gpurun_out/r02_pytest11.log
timeout 900 bash scripts/lib_ab.sh p11 "--config c2" base variants/old/libdquant_b200.so variants/teams1/libdquant_b200.so variants/ns_t1/libdquant_b200.so variants/fa1/libdquant_b200.so variants/t1fa1/libdquant_b200.so
for v in base eig1 eig2; do L=variants/$v/libdquant_b200.so; [ $v = base ] && L=""; DQ_LIB=$L timeout 300 python scripts/seal_cost.py --profile 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', {k[:40]:v for k,v in d['kernels_ms'].items() if 'eig' in k or 'jacobi' in k})"; done
