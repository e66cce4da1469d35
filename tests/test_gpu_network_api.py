"""The network-level drop-in (include/pg_network.h: build_network / forward /
infer / backward over host f64 tensors, network.cpp:308-480) against the f64
oracle on the same parameters and inputs: outputs, parameter gradients,
input gradients and BN running buffers within 1e-4 (max-norm relative per
tensor), in train and eval mode, for the c1 / c2 discriminator and generator."""
import ctypes as C

import numpy as np
import pytest

from paper_2102_10485_b200 import _native as N, baseline_arch
from parity import layer_tensors, rel_max

pytestmark = pytest.mark.gpu
_D = C.POINTER(C.c_double)


def _d(a):
    return a.ctypes.data_as(_D)


class Net:
    def __init__(self, spec, in_shape, seed, math):
        lib = N.lib()
        shp = (C.c_long * len(in_shape))(*in_shape)
        h = C.c_void_p()
        N.check(lib.pg_net_create(spec.encode(), shp, len(in_shape), seed, 0.02, math, 0, C.byref(h)), "pg_net_create")
        self.h, self.lib = h, lib
        self.np = lib.pg_net_param_count(h)
        self.nb = lib.pg_net_buffer_count(h)
        s, r = (C.c_long * 4)(), C.c_int()
        N.check(lib.pg_net_out_shape(h, s, C.byref(r)), "out_shape")
        self.out = tuple(s[:r.value])

    def params(self):
        p = np.zeros(self.np)
        N.check(self.lib.pg_net_get_params(self.h, _d(p)), "get_params")
        return p

    def buffers(self):
        b = np.zeros(max(self.nb, 1))
        N.check(self.lib.pg_net_get_buffers(self.h, _d(b)), "get_buffers")
        return b[:self.nb]

    def fwd_bwd(self, x, gy, train):
        B = x.shape[0]
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros((B,) + self.out)
        tr = C.c_void_p()
        N.check(self.lib.pg_net_forward(self.h, _d(x), B, 1 if train else 0, _d(y), C.byref(tr)), "forward")
        gp, gx = np.zeros(self.np), np.zeros(x.shape)
        gy = np.ascontiguousarray(gy, np.float64)
        N.check(self.lib.pg_net_backward(self.h, tr, _d(gy), B, _d(gp), _d(gx)), "backward")
        self.lib.pg_trace_destroy(tr)
        return y, gp, gx

    def close(self):
        self.lib.pg_net_destroy(self.h)


@pytest.mark.parametrize("math", [0, 1])
@pytest.mark.parametrize("cfg,net", [(1, "disc"), (1, "gen"), (2, "disc"), (2, "gen")])
@pytest.mark.parametrize("train", [True, False])
def test_network_api_matches_oracle(oracle, cfg, net, math, train):
    arch = baseline_arch(cfg)
    spec = arch.disc if net == "disc" else arch.gen
    in_shape = arch.image if net == "disc" else (arch.d_z,)
    dev = Net(spec, in_shape, 11, math)
    p0 = dev.params()
    # build_network's draws (network.cpp:308-343), cast to fp32
    ref_init = oracle.net_init(spec, " ".join(map(str, in_shape)), 11)
    assert rel_max(p0, ref_init) < 1e-7
    rng = np.random.default_rng(3)
    B = 6
    x = rng.uniform(-1, 1, (B,) + tuple(in_shape)) if net == "disc" else rng.normal(size=(B, arch.d_z))
    gy = rng.normal(size=(B,) + dev.out) / B
    y, gp, gx = dev.fwd_bwd(x, gy, train)
    ry, rgx, rgp, rbuf = oracle.net_fwd_bwd(64, spec, " ".join(map(str, in_shape)), p0, x, gy, train)
    assert rel_max(y.ravel(), ry) < 1e-4
    assert rel_max(gx.ravel(), rgx) < 1e-4
    for name, off, n, feeds_bn in layer_tensors(spec, in_shape):
        if feeds_bn and train:
            continue  # exact gradient 0 (BatchNorm removes the bias)
        sl = slice(off, off + n)
        assert rel_max(gp[sl], rgp[sl]) < 1e-4, name
    if train and dev.nb:
        assert rel_max(dev.buffers(), rbuf) < 1e-5
    dev.close()
