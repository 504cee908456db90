#!/bin/bash
# per-kernel launch list (ncu, serialised, cold-ish caches) of a short full bench run; tag = $1
TAG=${1:-x}
B32="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$B32 > gpurun_out/plain32_$TAG.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_attn|combine|tail_append|prepare" -c 200 --csv --log-file gpurun_out/launches_$TAG.csv $B32 > gpurun_out/ncu_launch_$TAG.log 2>&1
echo NCU=$?
python scripts/launch_summary.py gpurun_out/launches_$TAG.csv
