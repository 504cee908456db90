#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_attention.py -m gpu -q -x --timeout 900 -p no:cacheprovider -k "gqa or c5 or bf16 or graph or seal or tail_only" > gpurun_out/r02_pytest18.log 2>&1
echo PYTEST_RC=$? ; grep -E "FAILED|passed|failed|Error" gpurun_out/r02_pytest18.log | tail -5
timeout 900 bash scripts/lib_ab.sh p18 "--config c5" base variants/old/libdquant_b200.so
