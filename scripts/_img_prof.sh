#!/bin/bash
# ncu --set full of the c4 image-side GEMM kernels (conv1 fwd / dgrad / wgrad), exported as text
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/gemm_sweep.py --layers 1 --math tf32x3 --iters 1 > gpurun_out/img_plain.log 2>&1 || exit 1
for op in fwd wgrad dgrad; do
  timeout 600 ncu --set full --clock-control none --import-source on -s 3 -c 3 -o /tmp/img_$op \
    python scripts/gemm_sweep.py --layers 1 --math tf32x3 --iters 1 --ops $op > gpurun_out/img_ncu_$op.log 2>&1
  ncu -i /tmp/img_$op.ncu-rep --page details > gpurun_out/img_$op.details.txt 2>&1
  ncu -i /tmp/img_$op.ncu-rep --page raw --csv > gpurun_out/img_$op.raw.csv 2>&1
  gzip -f gpurun_out/img_$op.raw.csv
done
