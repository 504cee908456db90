#!/bin/bash
# round-2 evidence (one B200): bench lines C2-C5 (+ tail 512, seal, reference arm), the C2 launch
# list, --set full captures of the split / prepare / combine kernels and of the seal kernels.
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline"
for c in c2 c3 c4 c5; do timeout 900 $B --config $c > gpurun_out/r02f_$c.json 2> gpurun_out/r02f_$c.err; echo "$c rc=$?"; done
timeout 900 $B --tail 512 > gpurun_out/r02f_c2_tail512.json 2>/dev/null; echo tail rc=$?
timeout 900 $B --seal > gpurun_out/r02f_c2_seal.json 2>/dev/null; echo seal rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_ref.json 2>/dev/null; echo ref rc=$?
timeout 900 python bench.py > gpurun_out/r02f_c2_default.json 2>/dev/null; echo default rc=$?
bash scripts/launches.sh r02 > gpurun_out/r02_launches.log 2>&1; tail -5 gpurun_out/r02_launches.log
S="python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu-baseline"
$S > /dev/null 2>&1
for K in decode_attn attn_prepare combine; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 -o gpurun_out/r02_prof_$K $S > gpurun_out/r02_ncu_$K.log 2>&1; echo "$K NCU=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gram128|eig_tql|project128|quantize_tile16" -s 4 -c 5 -o gpurun_out/r02_prof_k3 python scripts/seal_cost.py --units 512 --reps 1 > gpurun_out/r02_ncu_k3.log 2>&1; echo K3 NCU=$?
