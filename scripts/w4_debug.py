"""Diagnostics for wgrad4.cu (PG_W4_DBG modes) on a tiny conv1 weight gradient."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2102_10485_b200 import _native as N
L, B, H = 1, 1, 8
oh = H // 2
d = N.ConvDesc(B=B, Cin=3, H=H, W=H, Cout=64, OH=oh, OW=oh, k=4, s=2, p=1)
g = torch.Generator().manual_seed(1)
x = torch.randn(L, B, H, H, 4, generator=g); x[..., 3] = 0
gy = torch.randn(L, B, oh, oh, 64, generator=g)
gw = torch.zeros(L, 64 * 16 * 4)
xd, gyd, gwd = x.cuda(), gy.cuda(), gw.cuda()
P = lambda t: C.c_void_p(t.data_ptr())
N.check(N.lib().pg_conv2d_bwd_filter(C.byref(d), L, P(xd), P(gyd), P(gwd), 64 * 64, 0, 1, None))
out = gwd.cpu().numpy().reshape(64, 16, 4)
dbg = int(os.environ.get("PG_W4_DBG", "0"))
xn, gn = x.numpy()[0, 0], gy.numpy()[0, 0]
ref = np.zeros((64, 16, 4))
for i in range(oh):
    for j in range(oh):
        for t in range(16):
            iy, ix = 2 * i - 1 + t // 4, 2 * j - 1 + t % 4
            xv = xn[iy, ix] if 0 <= iy < H and 0 <= ix < H else np.zeros(4)
            if dbg >= 2: xv = np.ones(4)
            gv = gn[i, j] if dbg < 3 else np.ones(64)
            ref[:, t, :] += np.outer(gv, xv)
if dbg == 1:
    print("dbg1 out[0:2,0,:]", out[0:2, 0, :], "out[63,15,:]", out[63, 15, :])
else:
    print(f"dbg{dbg}: max|out-ref|={np.abs(out-ref).max():.3e} max|ref|={np.abs(ref).max():.3e}")
    print(" out[0,:2,:]", out[0, :2, :].ravel(), "\n ref[0,:2,:]", ref[0, :2, :].ravel())
    nz = np.argwhere(np.abs(out) > 0)
    print(" nonzero count", len(nz), nz[:5].tolist())
