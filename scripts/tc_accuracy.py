"""Accuracy probe: dense FPROP through the C-ABI for several K, each math mode
vs a float64 numpy reference (max |err| / max |ref|, and the mean signed
error / max|ref| to expose biased (truncating) accumulation)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2102_10485_b200 import _native as N

lib = N.lib()


def ptr(t):
    return C.c_void_p(t.data_ptr())


rng = np.random.default_rng(1)
for K in (64, 512, 4096, 16384):
    L, B, nout = 1, 256, 128
    x = rng.normal(size=(L, B, K)).astype(np.float32)
    w = rng.normal(size=(L, nout, K)).astype(np.float32)
    ref = np.einsum("lbk,lok->lbo", x.astype(np.float64), w.astype(np.float64))
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    line = [f"K={K:6d}"]
    for math, name in ((0, "simt"), (1, "tf32x3"), (2, "tf32")):
        y = torch.zeros((L, B, nout), device="cuda")
        N.check(lib.pg_dense_fwd(L, B, K, nout, ptr(xd), ptr(wd), nout * K, None, 0, 0, 0.0, ptr(y), math, None))
        torch.cuda.synchronize()
        got = y.cpu().numpy().astype(np.float64)
        scale = np.abs(ref).max()
        line.append(f"{name}: max {np.abs(got - ref).max() / scale:.2e} bias {(got - ref).mean() / scale:+.1e}")
    print("  ".join(line), flush=True)
