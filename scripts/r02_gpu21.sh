#!/bin/bash
# GQA item timeline (cross-item schedule): base, softmax sub-phases, no fold, no UMMAs
mkdir -p gpurun_out
export G=8 UNITS=512 T=16384
echo "== base"; timeout 300 python scripts/attn_trace.py
echo "== smtrace"; SMTRACE=1 DQ_LIB=variants/smtrace/libdquant_b200.so timeout 300 python scripts/attn_trace.py
echo "== nullfold"; DQ_LIB=variants/nullfold/libdquant_b200.so timeout 300 python scripts/attn_trace.py
echo "== nullmma"; DQ_LIB=variants/nullmma/libdquant_b200.so timeout 300 python scripts/attn_trace.py
