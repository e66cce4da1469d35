#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/gemm_sweep.py --layers 1 --math tf32x3 --ops fwd --iters 1 > gpurun_out/plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 2 -c 1 -o /tmp/f4p python scripts/gemm_sweep.py --layers 1 --math tf32x3 --ops fwd --iters 1 > gpurun_out/f4p_ncu.log 2>&1
ncu -i /tmp/f4p.ncu-rep --page details > gpurun_out/f4p.details.txt 2>&1
ncu -i /tmp/f4p.ncu-rep --page source --csv --print-source sass > gpurun_out/f4p.sass.csv 2>&1; gzip -f gpurun_out/f4p.sass.csv
