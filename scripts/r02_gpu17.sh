#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_attention.py tests/test_gpu_kvcache.py tests/test_gpu_sharding.py tests/test_gpu_model.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/r02_pytest17.log 2>&1
echo PYTEST_RC=$? ; grep -E "FAILED|passed|failed|Error" gpurun_out/r02_pytest17.log | tail -5
timeout 900 bash scripts/lib_ab.sh p17 "--config c2" base variants/noinw/libdquant_b200.so
DQ_LIB=variants/trace/libdquant_b200.so timeout 300 python scripts/team_trace.py
timeout 600 python bench.py --model 7b --steps 10 --warmup 3 > gpurun_out/r02_model7b.json 2> gpurun_out/r02_model7b.err; echo MODEL_RC=$?; cat gpurun_out/r02_model7b.json | head -c 1500; tail -3 gpurun_out/r02_model7b.err
