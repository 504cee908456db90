#!/bin/bash
# re-entry baseline: full GPU suite, bench lines C1-C5 + default, C5 launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/r02_g30_tests.log 2>&1; echo TESTS=$?
tail -3 gpurun_out/r02_g30_tests.log
timeout 300 python bench.py > gpurun_out/r02_g30_default.json 2> gpurun_out/r02_g30_default.err; echo DEFAULT=$?
cat gpurun_out/r02_g30_default.json
for c in c1 c3 c4 c5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02_g30_$c.json 2> gpurun_out/r02_g30_$c.err; echo $c=$?
  python -c "import json,sys; d=json.load(open(sys.argv[1])); r=d.get('roofline',{}); print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('launch_ms'), r.get('frac'))" gpurun_out/r02_g30_$c.json
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02_g30_launches_c5.csv python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_g30_ncu_c5.log 2>&1; echo NCU=$?
