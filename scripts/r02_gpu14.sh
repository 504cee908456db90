#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02_pytest14.log 2>&1
echo PYTEST_RC=$? ; tail -4 gpurun_out/r02_pytest14.log
timeout 300 python scripts/seal_cost.py --profile > gpurun_out/r02_seal14.json 2>&1; tail -1 gpurun_out/r02_seal14.json
timeout 600 python bench.py --config c1 --steps 10 --warmup 2 > gpurun_out/r02_bench_c1.json 2> gpurun_out/r02_bench_c1.err; echo C1_RC=$?; cat gpurun_out/r02_bench_c1.json; tail -3 gpurun_out/r02_bench_c1.err
DQ_LIB=variants/trace/libdquant_b200.so timeout 300 python scripts/team_trace.py
timeout 900 bash scripts/lib_ab.sh p14 "--config c2" base variants/old/libdquant_b200.so
timeout 600 bash scripts/lib_ab.sh p14c3 "--config c3" base variants/old/libdquant_b200.so
