#!/bin/bash
# path 1 (tcgen05, g = 1) vs path 0 on C2 at HEAD; fresh ncu capture of the path-1 split kernel
mkdir -p gpurun_out
timeout 300 bash scripts/lib_ab.sh g57 "" base
timeout 300 bash scripts/lib_ab.sh g57tc "--tc 1" base
B="python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu-baseline --tc 1"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:decode_attn_tc -s 2 -c 1 -o gpurun_out/r02_prof_tc $B > /dev/null 2>&1; echo NCU=$?
