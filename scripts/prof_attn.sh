#!/bin/bash
# ncu evidence for the fused decode-attention kernel (run under gpurun, 1 GPU).
#   bash scripts/prof_attn.sh <tag>
TAG=${1:-v1}
B="python bench.py --layers 2 --steps 2 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 2 -c 1 -o gpurun_out/prof_attn_$TAG $B > gpurun_out/ncu_full_$TAG.log 2>&1
echo NCU_RC=$?
B32="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$B32 > gpurun_out/plain32_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_attn|combine|tail_append" -c 300 --csv --log-file gpurun_out/launches_$TAG.csv $B32 > gpurun_out/ncu_launch_$TAG.log 2>&1
echo NCU2_RC=$?
tail -3 gpurun_out/ncu_full_$TAG.log
