#!/bin/bash
# C3 (int2, 13B b32 8K) split-kernel anatomy: item timeline, memory-pipeline ceiling, no-contraction build
mkdir -p gpurun_out
export G=1 UNITS=1280 T=8192 BITS=2
echo "== trace"; DQ_LIB=variants/trace/libdquant_b200.so timeout 120 python scripts/attn_trace.py 2>&1 | tail -12
unset G UNITS T BITS
timeout 400 bash scripts/lib_ab.sh g56c3 "--config c3 --layers 8" base variants/nullstream/libdquant_b200.so variants/nullcons/libdquant_b200.so
timeout 400 bash scripts/lib_ab.sh g56c2 "--layers 8" base variants/nullstream/libdquant_b200.so variants/nullcons/libdquant_b200.so
