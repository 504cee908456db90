#!/bin/bash
# ncu evidence for one round (run under gpurun, 1 GPU): launch list of the full C2 bench
# and one --set full capture each of the split, prepare and combine kernels.
#   bash scripts/profile_round.sh <tag>
TAG=${1:-r01}
bash scripts/launches.sh $TAG
B="python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/plain_$TAG.log 2>&1 || exit 1
for K in decode_attn attn_prepare combine; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 -o gpurun_out/prof_${K}_$TAG $B \
    > gpurun_out/ncu_full_${K}_$TAG.log 2>&1
  echo "$K NCU=$?"
done
