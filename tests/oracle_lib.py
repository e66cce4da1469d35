"""Test-side binding of the CPU oracle (oracle/_build/liboracle.so).

Test infrastructure only: the oracle is the checker, never the thing measured.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
LIB = ORACLE_DIR / "_build" / "liboracle.so"
KAT = ORACLE_DIR / "_build" / "kat"

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists() or not KAT.exists():
            build()
        h = C.CDLL(str(LIB))
        P, D = C.c_void_p, C.POINTER(C.c_double)
        h.or_last_error.restype = C.c_char_p
        h.or_group_create.restype = P
        h.or_group_create.argtypes = [C.c_int, C.c_int, C.c_char_p, C.c_char_p, C.c_char_p, C.c_long, C.c_int, C.c_int,
                                      C.c_long, C.c_uint64, C.c_uint64, C.c_long, C.c_int, C.c_double, C.c_int]
        h.or_group_step.argtypes = [P, C.c_int, C.c_int]
        h.or_group_get.restype = C.c_long
        h.or_group_get.argtypes = [P, C.c_int, C.c_int, D, C.c_long]
        h.or_group_set.argtypes = [P, C.c_int, C.c_int, D, C.c_long]
        h.or_group_step_inputs.argtypes = [P, C.c_int, D, D, D, C.c_long, D]
        h.or_group_destroy.argtypes = [P]
        h.or_group_mixture.argtypes = [P, D, C.c_long, C.c_uint64, D, C.POINTER(C.c_int)]
        h.or_dataset_label.argtypes = [C.c_long, C.c_long, C.c_long, C.c_int, C.c_long, C.c_uint64, D]
        h.or_derive_seed.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
        h.or_partition.argtypes = [C.POINTER(C.c_int), C.c_long, C.c_int, C.POINTER(C.c_long), C.POINTER(C.c_long)]
        h.or_net_fwd_bwd.argtypes = [C.c_int, C.c_char_p, C.c_char_p, C.c_uint64, C.c_double, C.c_int, C.c_long, D, D, D,
                                     D, D, D, D]
        h.or_net_info.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_long), C.POINTER(C.c_long), C.POINTER(C.c_long)]
        h.or_net_init.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, C.c_double, D]
        h.or_group_set_masks.argtypes = [P, C.c_int, C.POINTER(C.c_uint8), C.c_long]
        h.or_group_mask_flips.restype = C.c_long
        h.or_group_mask_flips.argtypes = [P, C.c_int]
        h.or_group_record_masks.argtypes = [P, C.c_int]
        h.or_group_get_masks.restype = C.c_long
        h.or_group_get_masks.argtypes = [P, C.c_int, C.POINTER(C.c_uint8), C.c_long]
        h.or_bench_steps.restype = C.c_double
        h.or_bench_steps.argtypes = [C.c_int, C.c_int, C.c_int, C.c_long, C.c_int, C.c_int]
        _lib = h
    return _lib


def _d(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(lib().or_last_error().decode())


class OracleGroup:
    """Workers of one architecture for labels [first, first + n): the
    reference run_worker protocol on the cosine-field dataset."""

    def __init__(self, prec: int, cfg: int, n_labels: int, per_label: int, batch: int, first_label: int = 0,
                 data_seed: int = 1, base_seed: int = 1, epochs: int = 1, lr: float = 2e-4, threads: int = 8,
                 gen: str = "", disc: str = "", image: str = "", d_z: int = 100):
        h = lib().or_group_create(prec, cfg, gen.encode(), disc.encode(), image.encode(), d_z, n_labels, first_label,
                                  per_label, data_seed, base_seed, batch, epochs, lr, threads)
        if not h:
            raise RuntimeError(lib().or_last_error().decode())
        self.h = h
        self.n = n_labels

    def step(self, n: int = 1, threads: int = 8) -> None:
        check(lib().or_group_step(self.h, n, threads))

    def get(self, label: int, what: int) -> np.ndarray:
        n = lib().or_group_get(self.h, label, what, None, 0)
        if n < 0:
            raise RuntimeError(lib().or_last_error().decode())
        out = np.zeros(n, np.float64)
        lib().or_group_get(self.h, label, what, _d(out), n)
        return out

    def set(self, label: int, what: int, v: np.ndarray) -> None:
        v = np.ascontiguousarray(v, np.float64)
        check(lib().or_group_set(self.h, label, what, _d(v), v.size))

    def set_masks(self, label: int, masks: np.ndarray) -> None:
        """Force the ReLU / LeakyReLU masks of the label's next step (MaskTape,
        oracle.hpp): bytes in the order the step evaluates them."""
        m = np.ascontiguousarray(masks, np.uint8)
        self._keep = m
        check(lib().or_group_set_masks(self.h, label, m.ctypes.data_as(C.POINTER(C.c_uint8)), m.size))

    def mask_flips(self, label: int) -> int:
        """elements of the last taped step where the forced mask disagreed with the oracle's sign test"""
        return int(lib().or_group_mask_flips(self.h, label))

    def record_masks(self, label: int) -> None:
        """record the label's next step's own ReLU / LeakyReLU masks (MaskTape order)"""
        check(lib().or_group_record_masks(self.h, label))

    def recorded_masks(self, label: int) -> np.ndarray:
        n = lib().or_group_get_masks(self.h, label, None, 0)
        out = np.zeros(max(n, 0), np.uint8)
        if n > 0:
            lib().or_group_get_masks(self.h, label, out.ctypes.data_as(C.POINTER(C.c_uint8)), n)
        return out

    def mixture(self, priors, n: int, seed: int, sample_shape) -> tuple[np.ndarray, np.ndarray]:
        """mixture_sample (partition.cpp:182-227) over the group's pairs: samples in [0,1], class indices."""
        pri = np.ascontiguousarray(priors, np.float64)
        out = np.zeros((n, *sample_shape), np.float64)
        ids = np.zeros(n, np.int32)
        check(lib().or_group_mixture(self.h, _d(pri), n, seed, _d(out), ids.ctypes.data_as(C.POINTER(C.c_int))))
        return out, ids

    def step_inputs(self, label: int, real01: np.ndarray, z1: np.ndarray, z2: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(real01, np.float64)
        a = np.ascontiguousarray(z1, np.float64)
        b = np.ascontiguousarray(z2, np.float64)
        rep = np.zeros(4, np.float64)
        check(lib().or_group_step_inputs(self.h, label, _d(r), _d(a), _d(b), r.shape[0], _d(rep)))
        return rep

    def close(self) -> None:
        if self.h:
            lib().or_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dataset_label(shape, per_label: int, seed: int, label: int) -> np.ndarray:
    c, h, w = shape
    out = np.zeros((per_label, c, h, w), np.float64)
    check(lib().or_dataset_label(c, h, w, label, per_label, seed, _d(out)))
    return out


def derive_seed(base: int, stream: int) -> int:
    o = C.c_uint64()
    lib().or_derive_seed(base, stream, C.byref(o))
    return o.value


def net_info(spec: str, in_shape: str):
    p, b, o = C.c_long(), C.c_long(), C.c_long()
    check(lib().or_net_info(spec.encode(), in_shape.encode(), C.byref(p), C.byref(b), C.byref(o)))
    return p.value, b.value, o.value


def net_init(spec: str, in_shape: str, seed: int, init_std: float = 0.02) -> np.ndarray:
    n, _, _ = net_info(spec, in_shape)
    out = np.zeros(n, np.float64)
    check(lib().or_net_init(spec.encode(), in_shape.encode(), seed, init_std, _d(out)))
    return out


def net_fwd_bwd(prec: int, spec: str, in_shape: str, params: np.ndarray, x: np.ndarray, gy: np.ndarray | None,
                train: bool):
    """One forward (+ backward) of a layer list on given params; returns
    (y, gx, gparams, buffers_after)."""
    n_p, n_b, n_out = net_info(spec, in_shape)
    n = x.shape[0]
    x = np.ascontiguousarray(x, np.float64)
    params = np.ascontiguousarray(params, np.float64)
    y = np.zeros(n * n_out, np.float64)
    gx = np.zeros(x.size, np.float64)
    gp = np.zeros(n_p, np.float64)
    bufs = np.zeros(max(n_b, 1), np.float64)
    gyp = None if gy is None else _d(np.ascontiguousarray(gy, np.float64))
    keep = None if gy is None else np.ascontiguousarray(gy, np.float64)
    if keep is not None:
        gyp = _d(keep)
    check(lib().or_net_fwd_bwd(prec, spec.encode(), in_shape.encode(), 1, 0.02, 1 if train else 0, n, _d(x), gyp,
                               _d(params), _d(y), _d(gx), _d(gp), _d(bufs)))
    return y, gx, gp, bufs[:n_b]
