cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "conv2d or convT2d" -p no:cacheprovider 2>&1 | tail -2) > gpurun_out/f4_tests.log
for v in 0 1; do PG_FPROP4=$v timeout 300 python scripts/gemm_bench.py --op conv_fwd --layer 1 --iters 20 --save gpurun_out/f4_$v.npy; done > gpurun_out/f4_bench.log 2>&1
python scripts/ab_compare.py gpurun_out/f4_1.npy gpurun_out/f4_0.npy >> gpurun_out/f4_bench.log 2>&1
rm -f gpurun_out/*.npy
cat gpurun_out/f4_tests.log gpurun_out/f4_bench.log
