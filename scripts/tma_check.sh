#!/bin/bash
# TMA engine check: conv/convT kernel parity, then per-op timings TMA vs cp.async engine.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "conv" -p no:cacheprovider > gpurun_out/tma_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/tma_pytest.log
: > gpurun_out/tma_gb.log
for op in conv_fwd conv_dgrad conv_wgrad; do for layer in 2 3 4; do
  timeout 120 python scripts/gemm_bench.py --op $op --layer $layer --iters 3 >> gpurun_out/tma_gb.log 2>&1
  PG_NO_TMA=1 timeout 120 python scripts/gemm_bench.py --op $op --layer $layer --iters 3 2>&1 | sed 's/^/[cp.async] /' >> gpurun_out/tma_gb.log
done; done
tail -5 gpurun_out/tma_pytest.log; cat gpurun_out/tma_gb.log
