#!/bin/bash
# C5: does TMEM traffic from the Y loads slow the widening? widening span with / without Y loads / fold
mkdir -p gpurun_out
export G=8 UNITS=512 T=16384
for v in wt nullyld_wt nullfold_wt; do echo "== $v"; WIDETRACE=1 DQ_LIB=variants/$v/libdquant_b200.so timeout 60 python scripts/attn_trace.py 2>&1 | head -3; done
echo "== nullyld"; DQ_LIB=variants/nullyld/libdquant_b200.so timeout 60 python scripts/attn_trace.py 2>&1 | head -7
