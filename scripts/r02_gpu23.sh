#!/bin/bash
# GQA: widening with loads hoisted; MMA-warp sleep variant; traces
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -q -x -m gpu -k "gqa or c5" > gpurun_out/r02_g23_tests.log 2>&1; echo TESTS=$?
export G=8 UNITS=512 T=16384
echo "== widetrace"; WIDETRACE=1 DQ_LIB=variants/widetrace/libdquant_b200.so timeout 300 python scripts/attn_trace.py 2>&1 | head -5
echo "== mmawait"; MMAWAIT=1 DQ_LIB=variants/mmawait/libdquant_b200.so timeout 300 python scripts/attn_trace.py 2>&1 | head -3
unset G UNITS T
timeout 900 bash scripts/lib_ab.sh g23 "--config c5" base variants/mmasleep/libdquant_b200.so variants/gq_old/libdquant_b200.so
