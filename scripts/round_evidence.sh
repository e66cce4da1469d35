#!/bin/bash
# Full GPU evidence run for profiles/: default bench line, ncu launch list
# (time + DRAM bytes per launch) of a short bench, and a text export of one
# ncu --set full capture of the dominant implicit-GEMM kernel class.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_default.log
SHORT="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --gather-samples 8"
timeout 600 $SHORT > gpurun_out/bench_short.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launches.log
for spec in "conv_dgrad 2 gemm_pair" "conv_fwd 2 gemm_pair" "conv_wgrad 2 gemm_pair" "conv_fwd 1 fprop4" "conv_wgrad 1 wgrad4" "conv_dgrad 1 dgrad4"; do
  set -- $spec
  bash scripts/ncu_text.sh top_$1_$2 $3 python scripts/gemm_bench.py --op $1 --layer $2 --iters 1
done
tail -c 2500 gpurun_out/bench_default.log; tail -1 gpurun_out/ncu_launches.log
