"""Probe: tcgen05 engine vs SIMT engine on DGRAD / WGRAD / FPROP for one
descriptor variant (PG_TC_MN_VARIANT).  Prints max relative error per op."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2102_10485_b200 import _native as N
lib = N.lib()
def ptr(t): return C.c_void_p(t.data_ptr())
rng = np.random.default_rng(0)
L, B, nin, nout = 2, 40, 96, 64
x = torch.from_numpy(rng.normal(size=(L, B, nin)).astype(np.float32)).cuda()
w = torch.from_numpy(rng.normal(size=(L, nout * nin)).astype(np.float32)).cuda()
gy = torch.from_numpy(rng.normal(size=(L, B, nout)).astype(np.float32)).cuda()
res = {}
for math in (0, int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    y = torch.zeros((L, B, nout), device="cuda"); gx = torch.zeros((L, B, nin), device="cuda")
    gw = torch.zeros((L, nout * nin), device="cuda")
    N.check(lib.pg_dense_fwd(L, B, nin, nout, ptr(x), ptr(w), nout * nin, None, 0, 0, 0.0, ptr(y), math, None))
    N.check(lib.pg_dense_bwd_data(L, B, nin, nout, ptr(gy), ptr(w), nout * nin, ptr(gx), math, None))
    N.check(lib.pg_dense_bwd_filter(L, B, nin, nout, ptr(x), ptr(gy), ptr(gw), nout * nin, 0, math, None))
    torch.cuda.synchronize()
    res[math] = (y.cpu().numpy(), gx.cpu().numpy(), gw.cpu().numpy())
ref, got = res[0], res[max(res)]
for name, a, b in zip(("fprop", "dgrad", "wgrad"), got, ref):
    print(os.environ.get("PG_TC_MN_VARIANT", "0"), name, "%.3e" % (np.abs(a - b).max() / np.abs(b).max()))
