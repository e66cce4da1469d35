"""Compare two .npy outputs of scripts/gemm_bench.py --save (A/B of engine variants)."""
import sys
import numpy as np
a, b = np.load(sys.argv[1]).astype(np.float64), np.load(sys.argv[2]).astype(np.float64)
print(f"{sys.argv[1]} vs {sys.argv[2]}: max|a-b|/max|b| = {np.abs(a - b).max() / np.abs(b).max():.3e}")
