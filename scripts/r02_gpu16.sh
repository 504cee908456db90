#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02_pytest16.log 2>&1
echo PYTEST_RC=$? ; grep -E "FAILED|passed|failed" gpurun_out/r02_pytest16.log | tail -5
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo RC=$?
python -c "import json; d=json.load(open('gpurun_out/r02_bench_default.json')); print(d['value'], d['roofline'], d['e2e'], d['cpu_baseline'])"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
