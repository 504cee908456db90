#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02_pytest15.log 2>&1
echo PYTEST_RC=$? ; grep -E "FAILED|passed|failed" gpurun_out/r02_pytest15.log | tail -8
timeout 600 python bench.py --config c1 --steps 10 --warmup 2 > gpurun_out/r02_bench_c1b.json 2> gpurun_out/r02_bench_c1b.err; echo C1_RC=$?; cat gpurun_out/r02_bench_c1b.json | head -c 1500; echo; tail -3 gpurun_out/r02_bench_c1b.err
