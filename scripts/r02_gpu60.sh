#!/bin/bash
# GQA: Y in two head halves (N = 64 V UMMAs), the Y chain pipelined at half-stage granularity
mkdir -p gpurun_out
timeout 40 python -m pytest tests/test_gpu_attention.py -q -x -m gpu -k "test_gqa_tcgen05 and 4096" > gpurun_out/r02_g60_t0.log 2>&1; echo T0=$?
grep -q passed gpurun_out/r02_g60_t0.log || { tail -20 gpurun_out/r02_g60_t0.log; exit 3; }
timeout 300 python -m pytest tests/test_gpu_attention.py -q -x -m gpu -k "gqa or c5 or g8 or kernel_g or seal or step_graph" > gpurun_out/r02_g60_tests.log 2>&1; echo TESTS=$?
tail -2 gpurun_out/r02_g60_tests.log
export G=8 UNITS=512 T=16384
echo "== trace base"; timeout 60 python scripts/attn_trace.py 2>&1 | head -8
unset G UNITS T
timeout 300 bash scripts/lib_ab.sh g60 "--config c5 --layers 16" base variants/gq_old/libdquant_b200.so
