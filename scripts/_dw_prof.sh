#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/gemm_profile.py --labels 125 > gpurun_out/plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_wide -s 2 -c 2 -o /tmp/dw python scripts/gemm_profile.py --labels 125 > gpurun_out/dw_ncu.log 2>&1
ncu -i /tmp/dw.ncu-rep --page details > gpurun_out/dw.details.txt 2>&1
ncu -i /tmp/dw.ncu-rep --page source --csv --print-source sass > gpurun_out/dw.sass.csv 2>&1; gzip -f gpurun_out/dw.sass.csv
