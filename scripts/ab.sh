#!/bin/bash
# A/B kernel timing on one box: bench of the worktree ab_v8 (baseline) vs this tree
# usage: bash scripts/ab.sh <tag> [extra bench args for this tree...]
TAG=${1:-ab}; shift
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
get() { python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'ms/step', round(d['ms_per_step'],3), 'kernel_us', round(1e3*d['roofline']['launch_ms'],1), 'frac', round(d['roofline']['frac'],3))" $1 $2; }
for rep in 1 2; do
  (cd ab_v8 && $B > ../gpurun_out/ab_${TAG}_base$rep.json 2>/dev/null); get gpurun_out/ab_${TAG}_base$rep.json base$rep
  $B "$@" > gpurun_out/ab_${TAG}_new$rep.json 2>/dev/null; get gpurun_out/ab_${TAG}_new$rep.json new$rep
  $B --ctas 0 > gpurun_out/ab_${TAG}_c0$rep.json 2>/dev/null; get gpurun_out/ab_${TAG}_c0$rep.json c0_$rep
done
