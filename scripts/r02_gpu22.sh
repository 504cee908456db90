#!/bin/bash
# GQA role waits (cross-item schedule): MMA warp V phase, widening V stages (with and without the fold)
mkdir -p gpurun_out
export G=8 UNITS=512 T=16384
echo "== mmawait"; MMAWAIT=1 DQ_LIB=variants/mmawait/libdquant_b200.so timeout 300 python scripts/attn_trace.py 2>&1 | head -8
echo "== widetrace"; WIDETRACE=1 DQ_LIB=variants/widetrace/libdquant_b200.so timeout 300 python scripts/attn_trace.py 2>&1 | head -8
echo "== widenull"; WIDETRACE=1 DQ_LIB=variants/widenull/libdquant_b200.so timeout 300 python scripts/attn_trace.py 2>&1 | head -8
