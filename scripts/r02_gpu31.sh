#!/bin/bash
# C5 (GQA path 2) item timeline at HEAD: base, role waits, softmax sub-phases, spin / no-fold variants
mkdir -p gpurun_out
export G=8 UNITS=512 T=16384
echo "== base"; timeout 300 python scripts/attn_trace.py
echo "== mmawait"; MMAWAIT=1 DQ_LIB=variants/mmawait/libdquant_b200.so timeout 300 python scripts/attn_trace.py 2>&1 | head -4
echo "== widetrace"; WIDETRACE=1 DQ_LIB=variants/widetrace/libdquant_b200.so timeout 300 python scripts/attn_trace.py 2>&1 | head -4
echo "== smtrace"; SMTRACE=1 DQ_LIB=variants/smtrace/libdquant_b200.so timeout 300 python scripts/attn_trace.py 2>&1 | head -4
echo "== spin"; DQ_LIB=variants/spin/libdquant_b200.so timeout 300 python scripts/attn_trace.py 2>&1 | head -4
echo "== nullfold"; DQ_LIB=variants/nullfold/libdquant_b200.so timeout 300 python scripts/attn_trace.py 2>&1 | head -4
unset G UNITS T
timeout 900 bash scripts/lib_ab.sh g31 "--config c5 --layers 16" base variants/spin/libdquant_b200.so variants/nullfold/libdquant_b200.so
