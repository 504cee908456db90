#!/bin/bash
# one GPU iteration: parity tests, bench line, ncu of the attention kernel (tag = $1)
TAG=${1:-iter}
python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -4
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo BENCH_RC=$?
tail -2 gpurun_out/bench_$TAG.err
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json'))
print('value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'kernel_ms', round(d['roofline']['launch_ms'],4), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1))"
if [ "$2" == "ncu" ]; then
B="python bench.py --layers 2 --steps 2 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 2 -c 1 -o gpurun_out/prof_attn_$TAG $B > gpurun_out/ncu_full_$TAG.log 2>&1
echo NCU_RC=$?
fi
