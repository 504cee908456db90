#!/bin/bash
# round-2 GPU call 4: where the two-team kernel loses (null-stream A/B, ncu), seal kernels ncu
mkdir -p gpurun_out
timeout 600 bash scripts/lib_ab.sh ns "--config c2" base variants/ns_t2/libdquant_b200.so variants/ns_t1/libdquant_b200.so variants/teams1/libdquant_b200.so
B="python bench.py --layers 2 --steps 2 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/plain_t2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 2 -c 1 -o gpurun_out/r02_prof_t2 $B > gpurun_out/r02_ncu_t2.log 2>&1
echo NCU_RC=$?
S="python scripts/seal_cost.py --units 512 --reps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gram128|jacobi|project128|quantize_core" -s 4 -c 4 -o gpurun_out/r02_prof_seal $S > gpurun_out/r02_ncu_seal.log 2>&1
echo NCU2_RC=$?
