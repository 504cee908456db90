#!/bin/bash
# round-2 final measurements at HEAD: GPU suite, bench lines C1-C5 + model + reference arm,
# C5 launch list and one --set full capture of the GQA split kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/r02_g41_tests.log 2>&1; echo TESTS=$?
tail -2 gpurun_out/r02_g41_tests.log
timeout 300 python bench.py > gpurun_out/r02_g41_c2.json 2> gpurun_out/r02_g41_c2.err; echo C2=$?
for c in c1 c3 c4 c5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02_g41_$c.json 2> gpurun_out/r02_g41_$c.err; echo $c=$?
done
timeout 300 python bench.py --tail 512 --no-cpu-baseline > gpurun_out/r02_g41_c2_tail512.json 2>/dev/null; echo TAIL=$?
timeout 300 python bench.py --seal --no-cpu-baseline > gpurun_out/r02_g41_c2_seal.json 2>/dev/null; echo SEAL=$?
timeout 600 python bench.py --model 7b --steps 10 --warmup 3 > gpurun_out/r02_g41_model7b.json 2>/dev/null; echo M7B=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02_g41_ref.json 2>/dev/null; echo REF=$?
B5="python bench.py --config c5 --layers 2 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_g41_launches_c5.csv $B5 > gpurun_out/r02_g41_ncu_c5.log 2>&1; echo NCU5=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:decode_attn_gqa -s 2 -c 1 -o gpurun_out/r02_g41_prof_gqa $B5 > gpurun_out/r02_g41_ncu_gqa.log 2>&1; echo NCUFULL=$?
