#!/bin/bash
mkdir -p gpurun_out
timeout 900 bash scripts/lib_ab.sh p10 "--config c2" base variants/fa1/libdquant_b200.so variants/fa3/libdquant_b200.so variants/teams1/libdquant_b200.so variants/t1fa1/libdquant_b200.so
timeout 900 bash scripts/lib_ab.sh p10c4 "--config c4" base variants/fa1/libdquant_b200.so variants/t1fa1/libdquant_b200.so
