"""Micro-benchmark of one implicit-GEMM op of the c4 step through the C-ABI
(device-resident random data), CUDA-event timed; used for ncu captures.
  python scripts/gemm_bench.py --op conv_fwd --layer 2 [--math tf32x3] [--iters 5]
layers (c4 discriminator, 125 labels x batch 32): 1 = 3->64 64x64, 2 = 64->128 32x32,
3 = 128->256 16x16, 4 = 256->512 8x8; ops: conv_fwd, conv_dgrad, conv_wgrad, convt_fwd (the generator layer mirroring it)."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2102_10485_b200 import _native as N

p = argparse.ArgumentParser()
p.add_argument("--op", default="conv_fwd")
p.add_argument("--layer", type=int, default=2)
p.add_argument("--labels", type=int, default=125)
p.add_argument("--batch", type=int, default=32)
p.add_argument("--math", default="tf32x3")
p.add_argument("--iters", type=int, default=5)
p.add_argument("--save", default="", help="write the op output (.npy) for A/B comparisons")
args = p.parse_args()
math = {"fp32": 0, "tf32x3": 1, "tf32": 2}[args.math]
cin, cout, h = {1: (3, 64, 64), 2: (64, 128, 32), 3: (128, 256, 16), 4: (256, 512, 8)}[args.layer]
pad = lambda c: (c + 3) // 4 * 4
L, B = args.labels, args.batch
oh = h // 2
d = N.ConvDesc(B=B, Cin=cin, H=h, W=h, Cout=cout, OH=oh, OW=oh, k=4, s=2, p=1)
torch.manual_seed(0)
x = torch.randn(L, B, h, h, pad(cin), device="cuda")
gy = torch.randn(L, B, oh, oh, pad(cout), device="cuda")
wl = pad(cout) * 16 * pad(cin)
w = torch.randn(L, wl, device="cuda") * 0.02
bias = torch.zeros(L, pad(cout), device="cuda")
y = torch.empty(L, B, oh, oh, pad(cout), device="cuda")
gx = torch.empty_like(x)
gw = torch.empty_like(w)
dT = N.ConvDesc(B=B, Cin=cout, H=oh, W=oh, Cout=cin, OH=h, OW=h, k=4, s=2, p=1)
wT = torch.randn(L, wl, device="cuda") * 0.02
biasT = torch.zeros(L, pad(cin), device="cuda")
lib = N.lib()
P = lambda t: C.c_void_p(t.data_ptr())


def run():
    if args.op == "conv_fwd":
        N.check(lib.pg_conv2d_fwd(C.byref(d), L, P(x), P(w), wl, P(bias), pad(cout), 0, 0.0, P(y), math, None))
    elif args.op == "conv_dgrad":
        N.check(lib.pg_conv2d_bwd_data(C.byref(d), L, P(gy), P(w), wl, P(gx), math, None))
    elif args.op == "convt_fwd":  # the generator's mirror layer: cout -> cin channels, oh -> h (tanh on layer 1)
        N.check(lib.pg_convT2d_fwd(C.byref(dT), L, P(gy), P(wT), wl, P(biasT), pad(cin), 3 if args.layer == 1 else 1,
                                   0.0, P(gx), math, None))
    else:
        N.check(lib.pg_conv2d_bwd_filter(C.byref(d), L, P(x), P(gy), P(gw), wl, 0, math, None))


for _ in range(2):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.iters):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / args.iters
flops = 2.0 * L * B * oh * oh * cout * cin * 16
print(f"{args.op} layer {args.layer} ({cin}->{cout}, {h}x{h}) L={L} B={B} math={args.math}: {ms:.3f} ms, "
      f"{flops / ms / 1e9:.1f} TFLOP/s algorithmic")
if args.save:
    import numpy as np
    torch.manual_seed(0)
    out = {"conv_fwd": y, "conv_dgrad": gx, "convt_fwd": gx}.get(args.op, gw)
    np.save(args.save, out.cpu().numpy())
