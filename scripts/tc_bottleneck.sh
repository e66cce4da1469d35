#!/bin/bash
# time one step's GEMMs with parts of the tcgen05 kernel disabled (PG_TC_DEBUG bits)
for d in 0 1 2 3 4 8 12 15; do
  echo "== PG_TC_DEBUG=$d"
  PG_TC_DEBUG=$d timeout 300 python scripts/gemm_profile.py --labels 125 2>&1 | sed -n '1p;/fprop L=125 M=8192 N=128/{p;q}'
done
