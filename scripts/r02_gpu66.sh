#!/bin/bash
# C5: waits with __nanosleep back-off (math warps; + widening warps) against try_wait loops
mkdir -p gpurun_out
DQ_LIB=variants/nap2/libdquant_b200.so timeout 60 python -m pytest tests/test_gpu_attention.py -q -x -m gpu -k "test_gqa_tcgen05 and 4096" 2>&1 | tail -1
timeout 600 bash scripts/lib_ab.sh g66 "--config c5 --layers 16" base variants/nap1/libdquant_b200.so variants/nap2/libdquant_b200.so variants/nap1_256/libdquant_b200.so variants/nap2_32/libdquant_b200.so
