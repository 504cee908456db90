#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02_pytest12.log 2>&1
echo PYTEST_RC=$? ; tail -6 gpurun_out/r02_pytest12.log
timeout 600 python bench.py --seal --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_seal2.json 2> gpurun_out/r02_bench_seal2.err; echo SEAL_RC=$?
python -c "import json; d=json.load(open('gpurun_out/r02_bench_seal2.json')); print(d['seal'], d['ms_per_step'])"
tail -3 gpurun_out/r02_bench_seal2.err
DQ_LIB=variants/trace/libdquant_b200.so timeout 300 python scripts/team_trace.py
timeout 900 bash scripts/lib_ab.sh p12 "--config c2" base variants/ns_t1/libdquant_b200.so variants/t2/libdquant_b200.so
