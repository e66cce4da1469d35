#!/bin/bash
# ncu --set full of the three image-side (thin) conv kernels at the c4 shape.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for op in conv_fwd conv_dgrad conv_wgrad; do
  timeout 120 python scripts/gemm_bench.py --op $op --layer 1 --iters 3 >> gpurun_out/thin_gb.log 2>&1 && \
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:thin -s 1 -c 1 -o gpurun_out/prof_thin_$op \
     python scripts/gemm_bench.py --op $op --layer 1 --iters 1 > gpurun_out/ncu_thin_$op.log 2>&1
done
cat gpurun_out/thin_gb.log
