"""Kernel-level parity through the C-ABI (include/pg_kernels.h) against the
CPU oracle on identical seeded inputs, batched over several labels with
distinct weights.  Tolerances (per tensor, max|gpu-ref| / max|ref| vs the f64
oracle): FP32_SIMT and TF32X3 1e-5; TF32 (single pass, 10-bit mantissa) 5e-3;
BF16 (operands rounded to 8-bit significands) 2e-2 -- and, exactly, BF16 equals
an f64 GEMM of bf16-rounded operands to fp32 accumulation error
(test_bf16_mode_is_a_bf16_gemm).
"""
import ctypes as C

import numpy as np
import pytest

from parity import (conv_w_from_dev, conv_w_to_dev, convT_w_from_dev, convT_w_to_dev, nchw_to_nhwc, nhwc_to_nchw,
                    pad4, rel_max)

pytestmark = pytest.mark.gpu

MODES = [(0, 1e-5), (1, 1e-5), (2, 5e-3), (3, 2e-2)]  # BF16: operands rounded to 8-bit significands


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def ptr(t):
    return C.c_void_p(t.data_ptr())


def host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.float64)


CONV_CASES = [
    # (B, Cin, H, W, Cout, k, s, p)
    (2, 3, 8, 8, 8, 4, 2, 1),
    (3, 5, 7, 7, 6, 3, 2, 1),
    (2, 4, 6, 5, 4, 3, 1, 1),
    (2, 64, 8, 8, 128, 4, 2, 1),
    (2, 64, 16, 16, 256, 4, 2, 1),
    (16, 3, 32, 32, 64, 4, 2, 1),
    (4, 1, 28, 28, 64, 4, 2, 1),
    (4, 256, 8, 8, 512, 4, 2, 1),
    (4, 128, 16, 16, 256, 4, 2, 1),
    (4, 64, 32, 32, 128, 4, 2, 1),
    # TMA engine edge cases: padded 7x7 output boxes, batch not a multiple of the box depth
    (3, 64, 14, 14, 128, 4, 2, 1),
    (5, 128, 8, 8, 256, 4, 2, 1),
    (3, 32, 16, 16, 32, 4, 2, 1),
    # CTA-pair engine edge cases: odd number of M boxes (empty peer half), N not a multiple
    # of the pair tile (B half fully / partly out of bounds), WGRAD rows 16*Cin = 6 pair tiles
    (3, 64, 10, 10, 96, 4, 2, 1),
    (2, 96, 12, 12, 160, 4, 2, 1),
    # image side at the c4 shape (lowered im2col / column-GEMM + col2im paths)
    (4, 3, 64, 64, 64, 4, 2, 1),
]


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("math,tol", MODES)
def test_conv2d_fwd_bwd(native, oracle, torch_cuda, case, math, tol):
    from paper_2102_10485_b200 import _native as N
    torch = torch_cuda
    B, Cin, H, W, Cout, k, s, p = case
    L = 3
    OH, OW = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    spec = f"conv2d {Cin} {Cout} {k} {s} {p}"
    rng = np.random.default_rng(hash(case) % 2**32)
    nw = Cout * Cin * k * k
    wdev = np.zeros((L, pad4(Cout) * k * k * pad4(Cin)), np.float32)
    bias = np.zeros((L, pad4(Cout)), np.float32)
    xs, gys, refs = [], [], []
    for l in range(L):
        prm = rng.normal(0, 0.2, nw + Cout)
        x = rng.normal(0, 1, (B, Cin, H, W))
        gy = rng.normal(0, 1, (B, Cout, OH, OW))
        y, gx, gp, _ = oracle.net_fwd_bwd(64, spec, f"{Cin} {H} {W}", prm, x, gy, train=False)
        wdev[l] = conv_w_to_dev(prm[:nw].astype(np.float32), Cout, Cin, k).ravel()
        bias[l, :Cout] = prm[nw:]
        xs.append(nchw_to_nhwc(x.astype(np.float32)))
        gys.append(nchw_to_nhwc(gy.astype(np.float32)))
        refs.append((y.reshape(B, Cout, OH, OW), gx.reshape(B, Cin, H, W), gp))
    d = N.ConvDesc(B=B, Cin=Cin, H=H, W=W, Cout=Cout, OH=OH, OW=OW, k=k, s=s, p=p)
    x_d, gy_d = dev(torch, np.stack(xs)), dev(torch, np.stack(gys))
    w_d, b_d = dev(torch, wdev), dev(torch, bias)
    y_d = torch.zeros((L, B, OH, OW, pad4(Cout)), device="cuda")
    gx_d = torch.zeros((L, B, H, W, pad4(Cin)), device="cuda")
    gw_d = torch.full_like(w_d, 7.0)
    N.check(native.pg_conv2d_fwd(C.byref(d), L, ptr(x_d), ptr(w_d), wdev.shape[1], ptr(b_d), bias.shape[1], 0, 0.0,
                                 ptr(y_d), math, None), "fwd")
    N.check(native.pg_conv2d_bwd_data(C.byref(d), L, ptr(gy_d), ptr(w_d), wdev.shape[1], ptr(gx_d), math, None), "dgrad")
    N.check(native.pg_conv2d_bwd_filter(C.byref(d), L, ptr(x_d), ptr(gy_d), ptr(gw_d), wdev.shape[1], 0, math, None),
            "wgrad")
    y, gx, gw = host(y_d), host(gx_d), host(gw_d)
    for l in range(L):
        ry, rgx, rgp = refs[l]
        assert rel_max(nhwc_to_nchw(y[l], Cout), ry) < tol
        assert rel_max(nhwc_to_nchw(gx[l], Cin), rgx) < tol
        assert rel_max(conv_w_from_dev(gw[l], Cout, Cin, k), rgp[:nw].reshape(Cout, Cin, k, k)) < tol
        # padding stays exactly zero
        assert np.all(y[l][..., Cout:] == 0) and np.all(gx[l][..., Cin:] == 0)
    # accumulate mode adds
    N.check(native.pg_conv2d_bwd_filter(C.byref(d), L, ptr(x_d), ptr(gy_d), ptr(gw_d), wdev.shape[1], 1, math, None),
            "wgrad acc")
    assert rel_max(host(gw_d), 2 * gw) < 1e-6


CONVT_CASES = [
    (2, 8, 4, 4, 4, 4, 2, 1),
    (2, 5, 3, 3, 3, 4, 2, 1),
    (3, 4, 3, 4, 6, 3, 2, 1),
    (2, 6, 5, 5, 4, 3, 1, 1),
    (2, 128, 7, 7, 64, 4, 2, 1),
    (2, 256, 4, 4, 128, 4, 2, 1),
    (16, 64, 16, 16, 3, 4, 2, 1),
    (4, 64, 14, 14, 1, 4, 2, 1),
    (4, 512, 4, 4, 256, 4, 2, 1),
    (4, 256, 8, 8, 128, 4, 2, 1),
    (4, 128, 16, 16, 64, 4, 2, 1),
    (3, 256, 4, 4, 128, 4, 2, 1),
    (3, 64, 7, 7, 32, 4, 2, 1),
    (4, 64, 32, 32, 3, 4, 2, 1),
]


@pytest.mark.parametrize("case", CONVT_CASES)
@pytest.mark.parametrize("math,tol", MODES)
def test_convT2d_fwd_bwd(native, oracle, torch_cuda, case, math, tol):
    from paper_2102_10485_b200 import _native as N
    torch = torch_cuda
    B, Cin, H, W, Cout, k, s, p = case
    L = 2
    OH, OW = (H - 1) * s - 2 * p + k, (W - 1) * s - 2 * p + k
    spec = f"convT2d {Cin} {Cout} {k} {s} {p}"
    rng = np.random.default_rng(sum(case))
    nw = Cout * Cin * k * k
    wdev = np.zeros((L, pad4(Cin) * k * k * pad4(Cout)), np.float32)
    bias = np.zeros((L, pad4(Cout)), np.float32)
    xs, gys, refs = [], [], []
    for l in range(L):
        prm = rng.normal(0, 0.2, nw + Cout)
        x = rng.normal(0, 1, (B, Cin, H, W))
        gy = rng.normal(0, 1, (B, Cout, OH, OW))
        y, gx, gp, _ = oracle.net_fwd_bwd(64, spec, f"{Cin} {H} {W}", prm, x, gy, train=False)
        wdev[l] = convT_w_to_dev(prm[:nw].astype(np.float32), Cin, Cout, k).ravel()
        bias[l, :Cout] = prm[nw:]
        xs.append(nchw_to_nhwc(x.astype(np.float32)))
        gys.append(nchw_to_nhwc(gy.astype(np.float32)))
        refs.append((y.reshape(B, Cout, OH, OW), gx.reshape(B, Cin, H, W), gp))
    d = N.ConvDesc(B=B, Cin=Cin, H=H, W=W, Cout=Cout, OH=OH, OW=OW, k=k, s=s, p=p)
    x_d, gy_d = dev(torch, np.stack(xs)), dev(torch, np.stack(gys))
    w_d, b_d = dev(torch, wdev), dev(torch, bias)
    y_d = torch.zeros((L, B, OH, OW, pad4(Cout)), device="cuda")
    gx_d = torch.zeros((L, B, H, W, pad4(Cin)), device="cuda")
    gw_d = torch.zeros_like(w_d)
    N.check(native.pg_convT2d_fwd(C.byref(d), L, ptr(x_d), ptr(w_d), wdev.shape[1], ptr(b_d), bias.shape[1], 0, 0.0,
                                  ptr(y_d), math, None), "fwd")
    N.check(native.pg_convT2d_bwd_data(C.byref(d), L, ptr(gy_d), ptr(w_d), wdev.shape[1], ptr(gx_d), math, None),
            "dgrad")
    N.check(native.pg_convT2d_bwd_filter(C.byref(d), L, ptr(x_d), ptr(gy_d), ptr(gw_d), wdev.shape[1], 0, math, None),
            "wgrad")
    y, gx, gw = host(y_d), host(gx_d), host(gw_d)
    for l in range(L):
        ry, rgx, rgp = refs[l]
        assert rel_max(nhwc_to_nchw(y[l], Cout), ry) < tol
        assert rel_max(nhwc_to_nchw(gx[l], Cin), rgx) < tol
        assert rel_max(convT_w_from_dev(gw[l], Cin, Cout, k), rgp[:nw].reshape(Cin, Cout, k, k)) < tol


@pytest.mark.parametrize("dims", [(3, 64, 100, 6272), (2, 40, 6272, 4), (2, 300, 260, 200), (2, 16, 100, 4096),
                                  (2, 16, 4096, 1), (2, 4, 8192, 1), (2, 4, 100, 8192)])
@pytest.mark.parametrize("math,tol", MODES)
def test_dense_all_forms_multi_tile(native, torch_cuda, dims, math, tol):
    """Dense fwd / bwd-data / bwd-filter with several M and N tiles (e.g. the
    c1 generator head 100 -> 6272 and the discriminator head 6272 -> 1) vs an
    f64 numpy reference."""
    from paper_2102_10485_b200 import _native as N
    torch = torch_cuda
    L, B, nin, nout = dims
    rng = np.random.default_rng(nin + nout)
    x = rng.normal(size=(L, B, nin))
    w = rng.normal(size=(L, nout, nin)) * 0.05
    b = rng.normal(size=(L, nout))
    gy = rng.normal(size=(L, B, nout))
    pi, po = pad4(nin), pad4(nout)
    xd = np.zeros((L, B, pi), np.float32); xd[..., :nin] = x
    wd = np.zeros((L, po, pi), np.float32); wd[:, :nout, :nin] = w
    bd = np.zeros((L, po), np.float32); bd[:, :nout] = b
    gyd = np.zeros((L, B, po), np.float32); gyd[..., :nout] = gy
    x_d, w_d, b_d, gy_d = dev(torch, xd), dev(torch, wd), dev(torch, bd), dev(torch, gyd)
    y_d = torch.zeros((L, B, po), device="cuda")
    gx_d = torch.zeros((L, B, pi), device="cuda")
    gw_d = torch.zeros((L, po * pi), device="cuda")
    N.check(native.pg_dense_fwd(L, B, nin, nout, ptr(x_d), ptr(w_d), po * pi, ptr(b_d), po, 0, 0.0, ptr(y_d), math,
                                None), "fwd")
    N.check(native.pg_dense_bwd_data(L, B, nin, nout, ptr(gy_d), ptr(w_d), po * pi, ptr(gx_d), math, None), "dgrad")
    N.check(native.pg_dense_bwd_filter(L, B, nin, nout, ptr(x_d), ptr(gy_d), ptr(gw_d), po * pi, 0, math, None),
            "wgrad")
    y, gx, gw = host(y_d), host(gx_d), host(gw_d).reshape(L, po, pi)
    xf, wf, gyf = xd.astype(np.float64)[..., :nin], wd.astype(np.float64)[:, :nout, :nin], gyd.astype(np.float64)[..., :nout]
    for l in range(L):
        assert rel_max(y[l][:, :nout], xf[l] @ wf[l].T + bd[l, :nout]) < tol
        assert rel_max(gx[l][:, :nin], gyf[l] @ wf[l]) < tol
        assert rel_max(gw[l][:nout, :nin], gyf[l].T @ xf[l]) < tol


@pytest.mark.parametrize("math,tol", MODES)
def test_dense_fwd_bwd_with_activation(native, oracle, torch_cuda, math, tol):
    from paper_2102_10485_b200 import _native as N
    torch = torch_cuda
    L, B, nin, nout = 3, 5, 100, 36
    rng = np.random.default_rng(5)
    wdev = np.zeros((L, pad4(nout) * pad4(nin)), np.float32)
    bias = np.zeros((L, pad4(nout)), np.float32)
    xs, refs = [], []
    for l in range(L):
        prm = rng.normal(0, 0.2, nin * nout + nout)
        x = rng.normal(0, 1, (B, nin))
        y, _, _, _ = oracle.net_fwd_bwd(64, f"dense {nin} {nout}; lrelu 0.2", str(nin), prm, x, None, train=False)
        w = np.zeros((pad4(nout), pad4(nin)), np.float32)
        w[:nout, :nin] = prm[:nin * nout].reshape(nout, nin)
        wdev[l] = w.ravel()
        bias[l, :nout] = prm[nin * nout:]
        xs.append(x)
        refs.append(y.reshape(B, nout))
    x_d = dev(torch, np.stack(xs))
    w_d, b_d = dev(torch, wdev), dev(torch, bias)
    y_d = torch.zeros((L, B, pad4(nout)), device="cuda")
    N.check(native.pg_dense_fwd(L, B, nin, nout, ptr(x_d), ptr(w_d), wdev.shape[1], ptr(b_d), bias.shape[1],
                                N.ACT_LRELU, 0.2, ptr(y_d), math, None), "dense")
    y = host(y_d)
    for l in range(L):
        assert rel_max(y[l][:, :nout], refs[l]) < tol


@pytest.mark.parametrize("act,spec_act", [(1, "relu"), (2, "lrelu 0.2")])
@pytest.mark.parametrize("L,B,Cch,H,W", [(2, 6, 6, 5, 5), (2, 16, 128, 8, 8), (3, 40, 64, 7, 7), (2, 16, 256, 4, 4)])
def test_batchnorm_fwd_bwd_train(native, oracle, torch_cuda, act, spec_act, L, B, Cch, H, W):
    """BN over an NHWC map with the fused activation; statistics, running-stat
    update, dgamma/dbeta and the input gradient vs the oracle (1e-5).  Shapes
    cover one and several 512-row reduction chunks (ragged last chunk) and
    several labels."""
    from paper_2102_10485_b200 import _native as N
    torch = torch_cuda
    Cp = pad4(Cch)
    spec = f"bn {Cch}; {spec_act}"
    rng = np.random.default_rng(9)
    R = B * H * W
    xs, gys, gbs, runs, refs = [], [], [], [], []
    for l in range(L):
        prm = np.concatenate([rng.uniform(0.5, 1.5, Cch), rng.normal(0, 0.3, Cch)])
        x = rng.normal(0.3, 2.0, (B, Cch, H, W))
        gy = rng.normal(0, 1, (B, Cch, H, W))
        y, gx, gp, bufs = oracle.net_fwd_bwd(64, spec, f"{Cch} {H} {W}", prm, x, gy, train=True)
        xs.append(nchw_to_nhwc(x.astype(np.float32)))
        gys.append(nchw_to_nhwc(gy.astype(np.float32)))
        gbs.append(prm.astype(np.float32))
        run = np.concatenate([np.zeros(Cch), np.ones(Cch)]).astype(np.float32)
        runs.append(run)
        refs.append((y.reshape(B, Cch, H, W), gx.reshape(B, Cch, H, W), gp, bufs))
    x_d, gy_d = dev(torch, np.stack(xs)), dev(torch, np.stack(gys))
    gb_d, run_d = dev(torch, np.stack(gbs)), dev(torch, np.stack(runs))
    mean_d = torch.zeros((L, Cp), device="cuda")
    istd_d = torch.zeros((L, Cp), device="cuda")
    y_d = torch.zeros_like(x_d)
    gx_d = torch.zeros_like(x_d)
    dgb_d = torch.zeros((L, 2 * Cch), device="cuda")
    ws = torch.zeros(int(native.pg_bn_workspace_floats(L, R, Cp)), device="cuda")
    N.check(native.pg_bn_fwd(L, R, Cch, Cp, ptr(x_d), ptr(gb_d), 2 * Cch, ptr(run_d), 2 * Cch, 1e-5, 0.1, 1, act, 0.2,
                             ptr(mean_d), ptr(istd_d), ptr(y_d), ptr(ws), None), "bn fwd")
    N.check(native.pg_bn_bwd(L, R, Cch, Cp, ptr(gy_d), ptr(y_d), ptr(x_d), ptr(mean_d), ptr(istd_d), ptr(gb_d), 2 * Cch,
                             act, 0.2, ptr(gx_d), ptr(dgb_d), 2 * Cch, 0, ptr(ws), None), "bn bwd")
    y, gx, dgb, run = host(y_d), host(gx_d), host(dgb_d), host(run_d)
    for l in range(L):
        ry, rgx, rgp, rbuf = refs[l]
        assert rel_max(nhwc_to_nchw(y[l].reshape(B, H, W, Cp), Cch), ry) < 1e-5
        assert rel_max(nhwc_to_nchw(gx[l].reshape(B, H, W, Cp), Cch), rgx) < 1e-4
        assert rel_max(dgb[l], rgp) < 1e-5
        assert rel_max(run[l], rbuf) < 1e-5


def test_losses_and_clamp(native, torch_cuda):
    """gan.cpp:86-132 in f64 against a numpy restatement, incl. clamped entries."""
    from paper_2102_10485_b200 import _native as N
    torch = torch_cuda
    L, B, ps, c = 3, 7, 4, 1e-7
    rng = np.random.default_rng(2)
    pr = rng.uniform(0, 1, (L, B)).astype(np.float32)
    pf = rng.uniform(0, 1, (L, B)).astype(np.float32)
    pr[0, 0], pf[1, 2], pf[2, 3] = 1.0, 0.0, 1.0  # outside the clamp window
    P = np.zeros((L, B, ps), np.float32)
    Q = np.zeros((L, B, ps), np.float32)
    P[..., 0], Q[..., 0] = pr, pf
    pr_d, pf_d = dev(torch, P), dev(torch, Q)
    gr_d, gf_d, gg_d = torch.zeros_like(pr_d), torch.zeros_like(pr_d), torch.zeros_like(pr_d)
    rep = torch.zeros((L, 4), dtype=torch.float64, device="cuda")
    N.check(native.pg_gan_losses(L, B, ptr(pr_d), ptr(pf_d), ps, c, ptr(gr_d), ptr(gf_d), ptr(rep), None), "losses")
    N.check(native.pg_gen_loss(L, B, ptr(pf_d), ps, c, ptr(gg_d), ptr(rep), None), "gen loss")
    r = rep.cpu().numpy()
    gr, gf, gg = host(gr_d)[..., 0], host(gf_d)[..., 0], host(gg_d)[..., 0]
    for l in range(L):
        a, b = pr[l].astype(np.float64), pf[l].astype(np.float64)
        ca, cb = np.clip(a, c, 1 - c), np.clip(b, c, 1 - c)
        jd = -0.5 * np.log(ca).mean() - 0.5 * np.log(1 - cb).mean()
        jg = 0.5 * np.log(cb).mean()
        assert abs(r[l, 0] - jd) < 1e-12 * max(1, abs(jd))
        assert abs(r[l, 1] - jg) < 1e-12 * max(1, abs(jg))
        assert abs(r[l, 2] - a.mean()) < 1e-12 and abs(r[l, 3] - b.mean()) < 1e-12
        ins_a, ins_b = (a > c) & (a < 1 - c), (b > c) & (b < 1 - c)
        np.testing.assert_allclose(gr[l], np.where(ins_a, -0.5 / (B * a), 0), rtol=1e-6)
        np.testing.assert_allclose(gf[l], np.where(ins_b, 0.5 / (B * np.where(ins_b, 1 - b, 1)), 0), rtol=1e-6)
        np.testing.assert_allclose(gg[l], np.where(ins_b, -0.5 / (B * np.where(ins_b, b, 1)), 0), rtol=1e-6)
    assert gr[0, 0] == 0 and gf[1, 2] == 0 and gg[2, 3] == 0


def test_adam_matches_formula_and_rejects_nonfinite(native, torch_cuda):
    """optim.cpp:20-34 per label; a label with a NaN gradient is untouched."""
    from paper_2102_10485_b200 import _native as N
    torch = torch_cuda
    L, P = 3, 1024
    rng = np.random.default_rng(4)
    p0 = rng.normal(0, 0.02, (L, P)).astype(np.float32)
    p, m, v = p0.copy(), np.zeros_like(p0), np.zeros_like(p0)
    p_d, m_d, v_d = dev(torch, p), dev(torch, m), dev(torch, v)
    t_d = torch.zeros(L, dtype=torch.int64, device="cuda")
    f_d = torch.zeros(L, dtype=torch.int32, device="cuda")
    lr, b1, b2, eps = 2e-4, 0.5, 0.999, 1e-8
    for step in range(1, 6):
        g = rng.normal(0, 1e-3, (L, P)).astype(np.float32)
        if step == 3:
            g[1, 17] = np.nan
        g_d = dev(torch, g)
        N.check(native.pg_adam_step(L, P, ptr(p_d), ptr(g_d), ptr(m_d), ptr(v_d), ptr(t_d), ptr(f_d), lr, b1, b2, eps,
                                    None), "adam")
        for l in range(L):
            if l == 1 and step >= 3:
                continue
            # 1 - beta formed in f64 and rounded once (the kernel's ob1 / ob2)
            b1f, b2f, ob1, ob2 = np.float32(b1), np.float32(b2), np.float32(1 - b1), np.float32(1 - b2)
            m[l] = b1f * m[l] + ob1 * g[l]
            v[l] = b2f * v[l] + ob2 * g[l] * g[l]
            c1, c2 = np.float32(1 - b1 ** step), np.float32(1 - b2 ** step)
            p[l] = p[l] - np.float32(lr) * (m[l] / c1) / (np.sqrt(v[l] / c2) + np.float32(eps))
    assert host(f_d).tolist() == [0, 1, 0]
    assert host(t_d).tolist() == [5, 2, 5]
    np.testing.assert_allclose(host(p_d), p, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(host(m_d), m, rtol=1e-6, atol=1e-12)


def test_gather_real(native, torch_cuda):
    from paper_2102_10485_b200 import _native as N
    torch = torch_cuda
    L, n, B, H, W, Cc = 2, 9, 4, 3, 3, 3
    Cp = 4
    rng = np.random.default_rng(1)
    data = np.zeros((L, n, H, W, Cp), np.float32)
    data[..., :Cc] = rng.uniform(0, 1, (L, n, H, W, Cc))
    idx = rng.integers(0, n, (L, B)).astype(np.int32)
    d_d = dev(torch, data)
    i_d = torch.from_numpy(idx).cuda()
    o_d = torch.zeros((L, B, H, W, Cp), device="cuda")
    N.check(native.pg_gather_real(L, B, ptr(i_d), ptr(d_d), n * H * W * Cp, H * W * Cp, Cp, Cc, ptr(o_d), None), "gather")
    o = o_d.cpu().numpy()
    for l in range(L):
        want = data[l][idx[l]] * 2 - 1
        want[..., Cc:] = 0
        np.testing.assert_array_equal(o[l], want)


def test_caller_owned_workspace(native, torch_cuda):
    """pg_workspace_size / pg_set_workspace (the C-ABI never
    allocates): the image-side shapes that need scratch run bit-identically
    from a caller-owned buffer of exactly the reported size, and a buffer one
    256-byte granule short fails loudly."""
    torch = torch_cuda
    from paper_2102_10485_b200 import _native as N
    L, B = 2, 4
    d = N.ConvDesc(B=B, Cin=3, H=64, W=64, Cout=64, OH=32, OW=32, k=4, s=2, p=1)
    dT = N.ConvDesc(B=B, Cin=64, H=32, W=32, Cout=3, OH=64, OW=64, k=4, s=2, p=1)
    g = torch.Generator().manual_seed(5)
    big = torch.randn(L, B * 64 * 64 * 4, generator=g).cuda()
    small = torch.randn(L, B * 32 * 32 * 64, generator=g).cuda()
    w = (0.02 * torch.randn(L, 64 * 16 * 4, generator=g)).cuda()
    bias = torch.zeros(L, 4).cuda()
    runs = {
        N.PG_OP_CONV2D_BWD_FILTER: (d, lambda out: native.pg_conv2d_bwd_filter(
            C.byref(d), L, ptr(big), ptr(small), ptr(out), out.shape[1], 0, N.MATH_TF32X3, None), 64 * 16 * 4),
        N.PG_OP_CONVT2D_FWD: (dT, lambda out: native.pg_convT2d_fwd(
            C.byref(dT), L, ptr(small), ptr(w), w.shape[1], ptr(bias), 4, N.ACT_TANH, 0.0, ptr(out),
            N.MATH_TF32X3, None), B * 64 * 64 * 4),
        N.PG_OP_CONV2D_BWD_DATA: (d, lambda out: native.pg_conv2d_bwd_data(
            C.byref(d), L, ptr(small), ptr(w), w.shape[1], ptr(out), N.MATH_TF32X3, None), B * 64 * 64 * 4),
    }
    needs = {}
    try:
        for op, (desc, run, n_out) in runs.items():
            ref = torch.zeros(L, n_out).cuda()
            N.check(run(ref), "ws")
            need = native.pg_workspace_size(op, C.byref(desc), L, N.MATH_TF32X3)
            assert need < (1 << 40), (op, need)
            needs[op] = need
            if need == 0:  # this shape's engine takes no scratch (fprop4 / dgrad4 run in place)
                continue
            ws = torch.empty(need // 4 + 64, dtype=torch.float32, device="cuda")
            base = (ws.data_ptr() + 255) // 256 * 256
            N.check(native.pg_set_workspace(None, C.c_void_p(base), need), "ws")
            out = torch.zeros(L, n_out).cuda()
            N.check(run(out), "ws")
            torch.cuda.synchronize()
            assert torch.equal(out, ref), op
            N.check(native.pg_set_workspace(None, C.c_void_p(base), need - 256), "ws")
            rc = run(torch.zeros(L, n_out).cuda())
            assert rc == N.PG_EINVAL and b"workspace too small" in native.pg_last_error(), op
            N.check(native.pg_set_workspace(None, None, 0), "ws")
            del ws
        # the split-K weight gradient always takes scratch
        assert needs[N.PG_OP_CONV2D_BWD_FILTER] > 0, needs
    finally:
        native.pg_set_workspace(None, None, 0)


@pytest.mark.parametrize("math,tol", [(1, 1e-5), (2, 5e-3)])
def test_image_side_many_labels_per_cta(native, torch_cuda, math, tol):
    """The 4-channel image-side kernels (fprop4 / dgrad4 / wgrad4) walk a
    contiguous tile range per CTA and rebuild the label's weights on a label
    change; with 300 labels of one image each, every CTA crosses 2-3 labels.
    Checked per label against float64 torch (grouped conv = one label per
    group), including the generator's bias + tanh convT4 epilogue."""
    torch = torch_cuda
    import torch.nn.functional as F
    from paper_2102_10485_b200 import _native as N
    L, B, H = 300, 1, 64
    g = torch.Generator().manual_seed(11)
    x = torch.randn(L, B, 3, H, H, generator=g, dtype=torch.float64)
    w = 0.2 * torch.randn(L, 64, 3, 4, 4, generator=g, dtype=torch.float64)  # conv1: [Cout][Cin][k][k]
    b = 0.1 * torch.randn(L, 64, generator=g, dtype=torch.float64)
    gy = torch.randn(L, B, 64, H // 2, H // 2, generator=g, dtype=torch.float64)
    wt = 0.2 * torch.randn(L, 64, 3, 4, 4, generator=g, dtype=torch.float64)  # convT4: [Cin][Cout][k][k]
    bt = 0.1 * torch.randn(L, 3, generator=g, dtype=torch.float64)
    # float64 references, labels as groups
    xg = x.permute(1, 0, 2, 3, 4).reshape(B, L * 3, H, H)
    y_ref = F.conv2d(xg, w.reshape(L * 64, 3, 4, 4), b.reshape(-1), stride=2, padding=1, groups=L)
    gyg = gy.permute(1, 0, 2, 3, 4).reshape(B, L * 64, H // 2, H // 2)
    gx_ref = F.conv_transpose2d(gyg, w.reshape(L * 64, 3, 4, 4), stride=2, padding=1, groups=L)
    gw_ref = torch.stack([torch.nn.grad.conv2d_weight(x[l], w[l].shape, gy[l], stride=2, padding=1) for l in range(L)])
    pre_ref = F.conv_transpose2d(gyg, wt.reshape(L * 64, 3, 4, 4), bt.reshape(-1), stride=2, padding=1, groups=L)
    yt_ref = torch.tanh(pre_ref)

    def nhwc4(t):  # [L][B][C][h][w] -> [L][B][h][w][4] fp32 on the device
        out = torch.zeros(*t.shape[:2], t.shape[3], t.shape[4], 4, dtype=torch.float32)
        out[..., :t.shape[2]] = t.permute(0, 1, 3, 4, 2).float()
        return out.cuda()

    x_d = nhwc4(x)
    gy_d = gy.permute(0, 1, 3, 4, 2).float().contiguous().cuda()
    w_d = torch.zeros(L, 64, 16, 4)
    w_d[..., :3] = w.permute(0, 1, 3, 4, 2).reshape(L, 64, 16, 3).float()
    w_d = w_d.reshape(L, -1).cuda()
    wt_d = torch.zeros(L, 64, 16, 4)
    wt_d[..., :3] = wt.permute(0, 1, 3, 4, 2).reshape(L, 64, 16, 3).float()
    wt_d = wt_d.reshape(L, -1).cuda()
    b_d = b.float().cuda()
    bt_d = torch.zeros(L, 4)
    bt_d[:, :3] = bt.float()
    bt_d = bt_d.cuda()
    d = N.ConvDesc(B=B, Cin=3, H=H, W=H, Cout=64, OH=H // 2, OW=H // 2, k=4, s=2, p=1)
    dT = N.ConvDesc(B=B, Cin=64, H=H // 2, W=H // 2, Cout=3, OH=H, OW=H, k=4, s=2, p=1)
    y_d = torch.zeros(L, B, H // 2, H // 2, 64, device="cuda")
    gx_d = torch.zeros(L, B, H, H, 4, device="cuda")
    gw_d = torch.zeros_like(w_d)
    yt_d = torch.zeros(L, B, H, H, 4, device="cuda")
    N.check(native.pg_conv2d_fwd(C.byref(d), L, ptr(x_d), ptr(w_d), w_d.shape[1], ptr(b_d), 64, 0, 0.0, ptr(y_d),
                                 math, None), "fwd")
    N.check(native.pg_conv2d_bwd_data(C.byref(d), L, ptr(gy_d), ptr(w_d), w_d.shape[1], ptr(gx_d), math, None), "dgrad")
    N.check(native.pg_conv2d_bwd_filter(C.byref(d), L, ptr(x_d), ptr(gy_d), ptr(gw_d), w_d.shape[1], 0, math, None),
            "wgrad")
    N.check(native.pg_convT2d_fwd(C.byref(dT), L, ptr(gy_d), ptr(wt_d), wt_d.shape[1], ptr(bt_d), 4, N.ACT_TANH, 0.0,
                                  ptr(yt_d), math, None), "convT fwd")
    torch.cuda.synchronize()
    y = y_d.cpu().double().permute(0, 1, 4, 2, 3)  # [L][B][64][h][w]
    gx = gx_d.cpu().double()[..., :3].permute(0, 1, 4, 2, 3)
    gw = gw_d.cpu().double().reshape(L, 64, 4, 4, 4)[..., :3].permute(0, 1, 4, 2, 3)
    yt = yt_d.cpu().double()[..., :3].permute(0, 1, 4, 2, 3)
    y_ref = y_ref.reshape(B, L, 64, H // 2, H // 2).permute(1, 0, 2, 3, 4)
    gx_ref = gx_ref.reshape(B, L, 3, H, H).permute(1, 0, 2, 3, 4)
    yt_ref = yt_ref.reshape(B, L, 3, H, H).permute(1, 0, 2, 3, 4)
    pre_ref = pre_ref.reshape(B, L, 3, H, H).permute(1, 0, 2, 3, 4)
    worst = {}
    # tanh is 1-Lipschitz: its error is held to the tolerance of the pre-activation it saturates
    for name, got, ref, scale in (("fwd", y, y_ref, y_ref), ("dgrad", gx, gx_ref, gx_ref), ("wgrad", gw, gw_ref, gw_ref),
                                  ("convT", yt, yt_ref, pre_ref)):
        err = ((got - ref).abs().amax(dim=(1, 2, 3, 4)) / scale.abs().amax(dim=(1, 2, 3, 4))).max()
        worst[name] = float(err)
    assert max(worst.values()) < tol, worst
    assert torch.all(gx_d[..., 3] == 0) and torch.all(yt_d[..., 3] == 0)


def bf16_round(a):
    """numpy restatement of the device's nearest-even bfloat16 rounding (fp32 container)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


@pytest.mark.parametrize("case", [(4, 64, 16, 16, 128, 4, 2, 1), (4, 3, 64, 64, 64, 4, 2, 1), (2, 128, 8, 8, 256, 4, 2, 1)])
def test_bf16_mode_is_a_bf16_gemm(native, torch_cuda, case):
    """PG_MATH_BF16 on every conv GEMM form (forward, data and weight gradient;
    pair engine and the 4-channel image-side kernels) equals a float64
    convolution of the bf16-rounded operands up to fp32 accumulation error:
    the mode rounds both tensor-core operands and nothing else."""
    torch = torch_cuda
    import torch.nn.functional as F
    from paper_2102_10485_b200 import _native as N
    B, Cin, H, W, Cout, k, s, p = case
    L = 2
    OH, OW = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    rng = np.random.default_rng(5)
    x = rng.normal(0, 1, (L, B, Cin, H, W)).astype(np.float32)
    w = rng.normal(0, 0.2, (L, Cout, Cin, k, k)).astype(np.float32)
    gy = rng.normal(0, 1, (L, B, Cout, OH, OW)).astype(np.float32)
    xr, wr, gyr = (torch.from_numpy(bf16_round(a)).double() for a in (x, w, gy))
    y_ref = torch.stack([F.conv2d(xr[l], wr[l], stride=s, padding=p) for l in range(L)])
    gx_ref = torch.stack([F.conv_transpose2d(gyr[l], wr[l], stride=s, padding=p) for l in range(L)])
    gw_ref = torch.stack([torch.nn.grad.conv2d_weight(xr[l], wr[l].shape, gyr[l], stride=s, padding=p)
                          for l in range(L)])
    wdev = np.stack([conv_w_to_dev(w[l], Cout, Cin, k).ravel() for l in range(L)])
    x_d = dev(torch, np.stack([nchw_to_nhwc(x[l]) for l in range(L)]))
    gy_d = dev(torch, np.stack([nchw_to_nhwc(gy[l]) for l in range(L)]))
    w_d = dev(torch, wdev)
    b_d = torch.zeros((L, pad4(Cout)), device="cuda")
    y_d = torch.zeros((L, B, OH, OW, pad4(Cout)), device="cuda")
    gx_d = torch.zeros((L, B, H, W, pad4(Cin)), device="cuda")
    gw_d = torch.zeros_like(w_d)
    d = N.ConvDesc(B=B, Cin=Cin, H=H, W=W, Cout=Cout, OH=OH, OW=OW, k=k, s=s, p=p)
    N.check(native.pg_conv2d_fwd(C.byref(d), L, ptr(x_d), ptr(w_d), wdev.shape[1], ptr(b_d), pad4(Cout), 0, 0.0,
                                 ptr(y_d), N.MATH_BF16, None), "fwd")
    N.check(native.pg_conv2d_bwd_data(C.byref(d), L, ptr(gy_d), ptr(w_d), wdev.shape[1], ptr(gx_d), N.MATH_BF16,
                                      None), "dgrad")
    N.check(native.pg_conv2d_bwd_filter(C.byref(d), L, ptr(x_d), ptr(gy_d), ptr(gw_d), wdev.shape[1], 0,
                                        N.MATH_BF16, None), "wgrad")
    y, gx, gw = host(y_d), host(gx_d), host(gw_d)
    for l in range(L):
        assert rel_max(nhwc_to_nchw(y[l], Cout), y_ref[l].numpy()) < 1e-5
        assert rel_max(nhwc_to_nchw(gx[l], Cin), gx_ref[l].numpy()) < 1e-5
        assert rel_max(conv_w_from_dev(gw[l], Cout, Cin, k), gw_ref[l].numpy()) < 1e-5
