#!/bin/bash
# seal-cost diagnosis: --seal twice, then the launch list of a short --seal run (8 layers)
mkdir -p gpurun_out
for i in 1 2; do timeout 300 python bench.py --seal --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print(d['seal'])"; done
timeout 300 python bench.py --seal --layers 8 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print(d['seal'])"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_g42_launches_seal.csv python bench.py --seal --layers 8 --no-cpu-baseline > gpurun_out/r02_g42_ncu.log 2>&1; echo NCU=$?
python scripts/launch_summary.py gpurun_out/r02_g42_launches_seal.csv
timeout 300 python scripts/seal_cost.py 2>&1 | tail -15
