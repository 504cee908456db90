#!/bin/bash
# round-2 final state (after the step graphs): GPU suite, smoke, bench lines C1-C5 + model + reference arm
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/r02_g102_tests.log 2>&1; echo TESTS=$?
tail -2 gpurun_out/r02_g102_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo SMOKE=$?
timeout 300 python bench.py > gpurun_out/r02_g102_c2.json 2> gpurun_out/r02_g102_c2.err; echo C2=$?
timeout 300 python bench.py --config c1 > gpurun_out/r02_g102_c1.json 2>/dev/null; echo C1=$?
for c in c3 c4 c5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02_g102_$c.json 2>/dev/null; echo $c=$?
done
timeout 300 python bench.py --tail 512 --no-cpu-baseline > gpurun_out/r02_g102_c2_tail512.json 2>/dev/null; echo TAIL=$?
timeout 300 python bench.py --config c5 --tail 512 --no-cpu-baseline > gpurun_out/r02_g102_c5_tail512.json 2>/dev/null; echo TAIL5=$?
timeout 300 python bench.py --seal --no-cpu-baseline > gpurun_out/r02_g102_c2_seal.json 2>/dev/null; echo SEAL=$?
timeout 600 python bench.py --model 7b --steps 10 --warmup 3 > gpurun_out/r02_g102_model7b.json 2>/dev/null; echo M7B=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02_g102_ref.json 2>/dev/null; echo REF=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02_g102_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_g102_ncu_c2.log 2>&1; echo NCU=$?
