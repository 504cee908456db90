#!/bin/bash
# A/B of library variants on one box: bash scripts/lib_ab.sh <tag> "<bench args>" base variants/x/libdquant_b200.so ...
# ("base" = the in-tree library); two alternating repetitions, one summary line per run
TAG=$1; ARGS=$2; shift 2
get() { python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'ms/step', round(d['ms_per_step'],3), 'kernel_us', round(1e3*d['roofline']['launch_ms'],1), 'frac', round(d['roofline']['frac'],3), 'tok/s', round(d['value']))" $1 $2; }
for rep in 1 2; do
  for L in "$@"; do
    n=$(basename $(dirname $L)); [ "$L" = base ] && n=base
    out=gpurun_out/lab_${TAG}_${n}_$rep.json
    if [ "$L" = base ]; then python bench.py --steps 10 --warmup 3 --no-cpu-baseline $ARGS > $out 2>/dev/null
    else DQ_LIB=$L python bench.py --steps 10 --warmup 3 --no-cpu-baseline $ARGS > $out 2>/dev/null; fi
    get $out ${n}_$rep
  done
done
