"""Measured peaks of this B200 pool that are not in MEASURED_PEAKS.json (driver-written: HBM and
bf16 only).  FP64: scripts/fp64_rate.cu on a B200 of this pool (profiles/r02_fp64_rate.log):
DMMA (mma.sync.m8n8k4.f64) 37.1 TFLOP/s, DFMA 36.6 TFLOP/s."""

FP64_PEAK_TFLOPS = 37.1
