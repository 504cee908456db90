#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02_pytest13.log 2>&1
echo PYTEST_RC=$? ; tail -6 gpurun_out/r02_pytest13.log
DQ_LIB=variants/trace/libdquant_b200.so timeout 300 python scripts/team_trace.py
timeout 900 bash scripts/lib_ab.sh p13 "--config c2" base variants/old/libdquant_b200.so variants/ns_t1/libdquant_b200.so
for c in c3 c4 c5; do timeout 600 bash scripts/lib_ab.sh p13$c "--config $c" base variants/old/libdquant_b200.so; done
