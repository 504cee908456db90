#!/bin/bash
# round-2 GPU call 1: parity suite, C2 bench line, seal cost, K3 kernel launch list
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/r02_pytest1.log 2>&1
echo PYTEST_RC=$? ; tail -5 gpurun_out/r02_pytest1.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
echo BENCH_RC=$?; cat gpurun_out/r02_bench_c2.json | head -c 600; echo
python scripts/seal_cost.py --profile > gpurun_out/r02_seal.json 2>&1; echo SEAL_RC=$?; cat gpurun_out/r02_seal.json
python scripts/seal_cost.py --chunk 4096 --units 256 --profile > gpurun_out/r02_seal4k.json 2>&1; cat gpurun_out/r02_seal4k.json
