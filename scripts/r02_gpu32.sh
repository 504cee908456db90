#!/bin/bash
# TP harness: model tests (lock-step shards vs unsharded), whole-model 7B line at N=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_model.py -q -x > gpurun_out/r02_g32_model_tests.log 2>&1; echo TESTS=$?
tail -15 gpurun_out/r02_g32_model_tests.log
timeout 600 python bench.py --model 7b --steps 10 --warmup 3 > gpurun_out/r02_g32_model7b.json 2> gpurun_out/r02_g32_model7b.err; echo M7B=$?
cat gpurun_out/r02_g32_model7b.json; tail -5 gpurun_out/r02_g32_model7b.err
