#!/bin/bash
# Full GPU evidence run: tests, smoke, bench (default args), ncu launch list of
# a short bench, one ncu --set full capture of the top implicit-GEMM kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
SHORT="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --gather-samples 32"
timeout 600 $SHORT > gpurun_out/bench_short.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launches.log
timeout 600 python scripts/gemm_bench.py --op conv_fwd --layer 2 --iters 3 > gpurun_out/gb.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/prof_tc python scripts/gemm_bench.py --op conv_fwd --layer 2 --iters 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
tail -2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/ncu_launches.log gpurun_out/ncu_full.log; tail -c 3000 gpurun_out/bench.log
