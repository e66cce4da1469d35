#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/gemm_sweep.py --layers 1 --math tf32x3 --iters 1 --ops wgrad > gpurun_out/plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:thin_in_wgrad_mma -s 1 -c 1 -o /tmp/wg python scripts/gemm_sweep.py --layers 1 --math tf32x3 --iters 1 --ops wgrad > gpurun_out/wg_ncu.log 2>&1
ncu -i /tmp/wg.ncu-rep --page details > gpurun_out/wg.details.txt 2>&1
ncu -i /tmp/wg.ncu-rep --page source --csv --print-source sass > gpurun_out/wg.sass.csv 2>&1; gzip -f gpurun_out/wg.sass.csv
