"""Shared helpers for the GPU parity tests: reference <-> device layout
conversion and the tolerance metrics (documented in DESIGN.md §parity)."""
from __future__ import annotations

import numpy as np


def pad4(c: int) -> int:
    return (c + 3) // 4 * 4


def rel_max(a: np.ndarray, ref: np.ndarray) -> float:
    """max |a - ref| / max |ref| — per-tensor relative error (grads, outputs)."""
    a = np.asarray(a, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    scale = max(np.abs(ref).max(initial=0.0), 1e-30)
    return float(np.abs(a - ref).max(initial=0.0) / scale)


def rel_l2(a: np.ndarray, ref: np.ndarray) -> float:
    """||a - ref|| / ||ref|| — per-tensor relative error for updated weights
    (Adam's first steps are ~lr * sign(g), so a rare sign disagreement on a
    near-zero gradient moves one element by 2*lr; the L2 form weighs that
    by its share of the tensor)."""
    a = np.asarray(a, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    return float(np.linalg.norm(a - ref) / max(np.linalg.norm(ref), 1e-30))


def nchw_to_nhwc(x: np.ndarray, cp: int | None = None) -> np.ndarray:
    """[N][C][H][W] -> [N][H][W][Cp] with zero pad channels."""
    n, c, h, w = x.shape
    cp = cp or pad4(c)
    out = np.zeros((n, h, w, cp), x.dtype)
    out[..., :c] = x.transpose(0, 2, 3, 1)
    return out


def nhwc_to_nchw(x: np.ndarray, c: int) -> np.ndarray:
    return np.ascontiguousarray(x[..., :c].transpose(0, 3, 1, 2))


def conv_w_to_dev(w: np.ndarray, cout: int, cin: int, k: int) -> np.ndarray:
    """reference Conv2d weight [Cout][Cin][k][k] -> device [pad4(Cout)][k][k][pad4(Cin)]"""
    d = np.zeros((pad4(cout), k, k, pad4(cin)), w.dtype)
    d[:cout, :, :, :cin] = w.reshape(cout, cin, k, k).transpose(0, 2, 3, 1)
    return d


def conv_w_from_dev(d: np.ndarray, cout: int, cin: int, k: int) -> np.ndarray:
    return np.ascontiguousarray(d.reshape(pad4(cout), k, k, pad4(cin))[:cout, :, :, :cin].transpose(0, 3, 1, 2))


def convT_w_to_dev(w: np.ndarray, cin: int, cout: int, k: int) -> np.ndarray:
    """reference ConvTranspose2d weight [Cin][Cout][k][k] -> device [pad4(Cin)][k][k][pad4(Cout)]"""
    d = np.zeros((pad4(cin), k, k, pad4(cout)), w.dtype)
    d[:cin, :, :, :cout] = w.reshape(cin, cout, k, k).transpose(0, 2, 3, 1)
    return d


def convT_w_from_dev(d: np.ndarray, cin: int, cout: int, k: int) -> np.ndarray:
    return np.ascontiguousarray(d.reshape(pad4(cin), k, k, pad4(cout))[:cin, :, :, :cout].transpose(0, 3, 1, 2))


def layer_tensors(spec: str, in_shape: tuple) -> list[tuple[str, int, int, bool]]:
    """(name, offset, size, feeds_bn) of every parameter tensor of a layer
    list in the reference flat layout; feeds_bn marks a linear-layer bias
    followed by BatchNorm (its exact gradient is zero)."""
    items = [t.split() for t in spec.split(";") if t.split()]
    out, off = [], 0
    for i, tok in enumerate(items):
        nxt = [t[0] for t in items[i + 1:i + 2]]
        # a per-channel bias directly before BatchNorm is a gauge direction; a
        # dense bias reshaped to [C,H,W] is per position and is not
        feeds_bn = nxt == ["bn"]
        if tok[0] == "dense":
            a, b = int(tok[1]), int(tok[2])
            out += [(f"{i}.dense.w", off, a * b, False), (f"{i}.dense.b", off + a * b, b, feeds_bn)]
            off += a * b + b
        elif tok[0] in ("conv2d", "convT2d"):
            a, b, k = int(tok[1]), int(tok[2]), int(tok[3])
            n = a * b * k * k
            out += [(f"{i}.{tok[0]}.w", off, n, False), (f"{i}.{tok[0]}.b", off + n, b, feeds_bn)]
            off += n + b
        elif tok[0] == "bn":
            c = int(tok[1])
            out += [(f"{i}.bn.gamma", off, c, False), (f"{i}.bn.beta", off + c, c, False)]
            off += 2 * c
    return out


def update_err(p_new: np.ndarray, p_ref_new: np.ndarray, p_old: np.ndarray) -> float:
    """Error of an optimizer update (p_new - p_old vs p_ref_new - p_old) in
    units of the bar: max over elements of |du - dr| / (max|dr| + ulp32),
    i.e. relative to the largest reference update, with the fp32 rounding of
    the stored weight itself (one ulp of p_ref_new in float32) added to the
    allowance -- an fp32 parameter near 1 (BN gamma) cannot hold a 1e-4
    update to better than ~1e-3 of itself."""
    du = np.asarray(p_new, np.float64) - p_old
    dr = np.asarray(p_ref_new, np.float64) - p_old
    scale = max(np.abs(dr).max(initial=0.0), 1e-30)
    ulp = np.spacing(np.abs(p_ref_new).astype(np.float32)).astype(np.float64)
    return float((np.abs(du - dr) / (scale + ulp / 1e-4)).max(initial=0.0))
