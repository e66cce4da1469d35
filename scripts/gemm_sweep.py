"""Per-GEMM table of the c4 step's conv GEMMs through the C-ABI (device-resident
random data, CUDA events): every D conv layer x {fwd, dgrad, wgrad} x math
mode, with the algorithmic TFLOP/s.  ConvT layers of G are the same GEMMs with
roles swapped (convT fwd = conv dgrad, convT dgrad = conv fwd).
  python scripts/gemm_sweep.py [--labels 125] [--batch 32] [--iters 5] [--math tf32x3,tf32]"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2102_10485_b200 import _native as N

p = argparse.ArgumentParser()
p.add_argument("--labels", type=int, default=125)
p.add_argument("--batch", type=int, default=32)
p.add_argument("--iters", type=int, default=5)
p.add_argument("--math", default="tf32x3,tf32")
p.add_argument("--layers", default="1,2,3,4")
p.add_argument("--ops", default="fwd,dgrad,wgrad")
args = p.parse_args()
lib = N.lib()
P = lambda t: C.c_void_p(t.data_ptr())
pad = lambda c: (c + 3) // 4 * 4
L, B = args.labels, args.batch
print(f"L={L} B={B}")
print(f"{'layer':>16} {'op':>6} {'math':>7} {'ms':>8} {'TF/s':>7}")
for mname in args.math.split(","):
    math = {"fp32": 0, "tf32x3": 1, "tf32": 2}[mname]
    for layer in map(int, args.layers.split(",")):
        cin, cout, h = {1: (3, 64, 64), 2: (64, 128, 32), 3: (128, 256, 16), 4: (256, 512, 8)}[layer]
        oh = h // 2
        d = N.ConvDesc(B=B, Cin=cin, H=h, W=h, Cout=cout, OH=oh, OW=oh, k=4, s=2, p=1)
        x = torch.randn(L, B, h, h, pad(cin), device="cuda")
        gy = torch.randn(L, B, oh, oh, pad(cout), device="cuda")
        wl = pad(cout) * 16 * pad(cin)
        w = torch.randn(L, wl, device="cuda") * 0.02
        bias = torch.zeros(L, pad(cout), device="cuda")
        y = torch.empty(L, B, oh, oh, pad(cout), device="cuda")
        gx = torch.empty_like(x)
        gw = torch.empty_like(w)
        for op in args.ops.split(","):
            def run():
                if op == "fwd":
                    N.check(lib.pg_conv2d_fwd(C.byref(d), L, P(x), P(w), wl, P(bias), pad(cout), 0, 0.0, P(y), math,
                                              None))
                elif op == "dgrad":
                    N.check(lib.pg_conv2d_bwd_data(C.byref(d), L, P(gy), P(w), wl, P(gx), math, None))
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
            print(f"{f'{layer} {cin}->{cout} {h}x{h}':>16} {op:>6} {mname:>7} {ms:8.3f} {flops / ms / 1e9:7.1f}",
                  flush=True)
