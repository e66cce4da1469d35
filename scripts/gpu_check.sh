#!/bin/bash
# one gpurun call: env info, GPU tests, smoke, short bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{ nproc; lscpu | grep -E "Model name|Flags" | cut -c1-300; nvidia-smi -L; } > gpurun_out/env.log 2>&1
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -q -m gpu ${PYTEST_ARGS} --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout ${BENCH_TIMEOUT:-900} python bench.py ${BENCH_ARGS:---steps 2 --warmup 1 --no-cpu-baseline} > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/bench.log
