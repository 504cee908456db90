#!/bin/bash
# round-2 GPU call 9: ncu of the two-producer T2 kernel and the T1 build; vectorised segment tables
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -m gpu -q --timeout 600 -x -p no:cacheprovider > gpurun_out/r02_pytest9.log 2>&1
echo PYTEST_RC=$? ; tail -3 gpurun_out/r02_pytest9.log
B="python bench.py --layers 2 --steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 2 -c 1 -o gpurun_out/r02_prof_t2b $B > gpurun_out/r02_ncu_t2b.log 2>&1
echo NCU_RC=$?
DQ_LIB=variants/teams1/libdquant_b200.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 2 -c 1 -o gpurun_out/r02_prof_t1b $B > gpurun_out/r02_ncu_t1b.log 2>&1
echo NCU_RC=$?
timeout 600 python bench.py --seal --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_seal.json 2> gpurun_out/r02_bench_seal.err; echo SEAL_RC=$?
python -c "import json; d=json.load(open('gpurun_out/r02_bench_seal.json')); print(d['seal'], d['ms_per_step'])"
tail -3 gpurun_out/r02_bench_seal.err
