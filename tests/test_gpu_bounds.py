"""Out-of-bounds write checks for every GEMM engine through the C-ABI (the
pool's compute-sanitizer is closed): each operator writes into
the middle of a buffer whose 64 KB guard zones on both sides hold a NaN bit
pattern; after conv2d / convT2d / dense forward, data-gradient and weight
gradient (plain and accumulate) at the c4 layer shapes with a ragged batch,
every guard byte is unchanged and every read-only operand is bit-identical
to its upload.  Covers the CTA-pair engine (FPROP, DGRAD, phase-packed DGRAD,
WGRAD, the 4-channel F4 tiles), the lowered column-GEMM + col2im path, the thin
SIMT / mma.sync kernels and the dense latent-projection kernel."""
import ctypes as C

import numpy as np
import pytest

from parity import pad4

pytestmark = pytest.mark.gpu
GUARD = 16384  # floats per side
SENTINEL = np.frombuffer(np.uint32(0x7FC0DEAD).tobytes(), np.float32)[0]


class Guarded:
    """a device buffer of n floats between two sentinel-filled guard zones"""

    def __init__(self, torch, n, fill=None):
        self.buf = torch.full((n + 2 * GUARD,), float(SENTINEL), device="cuda")
        self.buf.view(torch.int32)[:] = 0x7FC0DEAD
        self.n = n
        self.t = self.buf[GUARD:GUARD + n]
        if fill is not None:
            self.t.copy_(torch.from_numpy(np.ascontiguousarray(fill, np.float32).ravel()).cuda())

    def ptr(self):
        return C.c_void_p(self.t.data_ptr())

    def guards_ok(self, torch):
        torch.cuda.synchronize()
        raw = self.buf.view(torch.int32).cpu().numpy()
        return bool(np.all(raw[:GUARD] == 0x7FC0DEAD) and np.all(raw[GUARD + self.n:] == 0x7FC0DEAD))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


LAYERS = [  # (Cin, Cout, H) of the c4 discriminator convs; convT = the generator's mirror images
    (3, 64, 64), (64, 128, 32), (128, 256, 16), (256, 512, 8)]


@pytest.mark.parametrize("math", [0, 1, 2])
@pytest.mark.parametrize("transposed", [False, True])
@pytest.mark.parametrize("layer", LAYERS)
def test_conv_ops_stay_in_bounds(native, torch_cuda, layer, transposed, math):
    from paper_2102_10485_b200 import _native as N
    torch = torch_cuda
    Cin, Cout, H = layer
    if transposed:  # generator layer Cout -> Cin at H/2 -> H
        cin, cout, h, oh = Cout, Cin, H // 2, H
    else:
        cin, cout, h, oh = Cin, Cout, H, H // 2
    L, B = 3, 5
    rng = np.random.default_rng(1)
    d = N.ConvDesc(B=B, Cin=cin, H=h, W=h, Cout=cout, OH=oh, OW=oh, k=4, s=2, p=1)
    xs = rng.normal(0, 1, (L, B, h, h, pad4(cin))).astype(np.float32)
    xs[..., cin:] = 0
    gys = rng.normal(0, 1, (L, B, oh, oh, pad4(cout))).astype(np.float32)
    gys[..., cout:] = 0
    wl = pad4(cin) * 16 * pad4(cout)
    w = (rng.normal(0, 0.05, (L, wl))).astype(np.float32)
    bias = rng.normal(0, 0.1, (L, pad4(cout))).astype(np.float32)
    x_g, gy_g, w_g, b_g = (Guarded(torch, a.size, a) for a in (xs, gys, w, bias))
    y_g = Guarded(torch, gys.size)
    gx_g = Guarded(torch, xs.size)
    gw_g = Guarded(torch, w.size, np.zeros_like(w))
    fwd, bwd_d, bwd_f = ((native.pg_convT2d_fwd, native.pg_convT2d_bwd_data, native.pg_convT2d_bwd_filter) if transposed
                         else (native.pg_conv2d_fwd, native.pg_conv2d_bwd_data, native.pg_conv2d_bwd_filter))
    N.check(fwd(C.byref(d), L, x_g.ptr(), w_g.ptr(), wl, b_g.ptr(), pad4(cout), 2, 0.2, y_g.ptr(), math, None), "fwd")
    N.check(bwd_d(C.byref(d), L, gy_g.ptr(), w_g.ptr(), wl, gx_g.ptr(), math, None), "dgrad")
    for acc in (0, 1):
        N.check(bwd_f(C.byref(d), L, x_g.ptr(), gy_g.ptr(), gw_g.ptr(), wl, acc, math, None), "wgrad")
    for name, g in (("y", y_g), ("gx", gx_g), ("gw", gw_g), ("x", x_g), ("gy", gy_g), ("w", w_g), ("bias", b_g)):
        assert g.guards_ok(torch), f"guard zone of {name} overwritten"
    for name, g, a in (("x", x_g, xs), ("gy", gy_g, gys), ("w", w_g, w), ("bias", b_g, bias)):
        assert np.array_equal(g.t.cpu().numpy().view(np.int32), a.ravel().view(np.int32)), f"read-only {name} modified"
    assert np.isfinite(y_g.t.cpu().numpy()).all() and np.isfinite(gx_g.t.cpu().numpy()).all()


@pytest.mark.parametrize("math", [0, 1, 2])
@pytest.mark.parametrize("shape", [(100, 8192), (8192, 1), (100, 6272), (4096, 1)])
def test_dense_ops_stay_in_bounds(native, torch_cuda, shape, math):
    from paper_2102_10485_b200 import _native as N
    torch = torch_cuda
    fin, fout = shape
    L, B = 3, 33
    rng = np.random.default_rng(2)
    x = rng.normal(0, 1, (L, B, pad4(fin))).astype(np.float32)
    x[..., fin:] = 0
    gy = rng.normal(0, 1, (L, B, pad4(fout))).astype(np.float32)
    gy[..., fout:] = 0
    w = rng.normal(0, 0.05, (L, pad4(fout) * pad4(fin))).astype(np.float32)
    b = rng.normal(0, 0.1, (L, pad4(fout))).astype(np.float32)
    x_g, gy_g, w_g, b_g = (Guarded(torch, a.size, a) for a in (x, gy, w, b))
    y_g, gx_g, gw_g = Guarded(torch, gy.size), Guarded(torch, x.size), Guarded(torch, w.size, np.zeros_like(w))
    N.check(native.pg_dense_fwd(L, B, fin, fout, x_g.ptr(), w_g.ptr(), w.shape[1], b_g.ptr(), b.shape[1], 1, 0.0,
                                y_g.ptr(), math, None), "dense fwd")
    N.check(native.pg_dense_bwd_data(L, B, fin, fout, gy_g.ptr(), w_g.ptr(), w.shape[1], gx_g.ptr(), math, None), "dgrad")
    for acc in (0, 1):
        N.check(native.pg_dense_bwd_filter(L, B, fin, fout, x_g.ptr(), gy_g.ptr(), gw_g.ptr(), w.shape[1], acc, math,
                                           None), "wgrad")
    for name, g in (("y", y_g), ("gx", gx_g), ("gw", gw_g), ("x", x_g), ("gy", gy_g), ("w", w_g), ("b", b_g)):
        assert g.guards_ok(torch), f"guard zone of {name} overwritten"
