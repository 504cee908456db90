#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --config c5 --layers 2 --steps 2 --warmup 3 --no-cpu-baseline"
$B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn_gqa -s 4 -c 1 -o gpurun_out/r02_prof_gqa $B > gpurun_out/r02_ncu_gqa.log 2>&1; echo NCU=$?
