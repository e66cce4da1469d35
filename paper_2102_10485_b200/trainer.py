"""Python face of the native trainer — mirrors the reference's
make_gan_pair / train_step / run_worker / generate for a *group* of labels
resident on one GPU (include/pg_trainer.h).  Arrays cross the boundary as
host numpy buffers; the device work happens inside the library.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .archs import Arch, baseline_arch


@dataclass
class StepReport:
    """gan.hpp:64-69"""
    j_d: float
    j_g: float
    d_real_mean: float
    d_fake_mean: float


@dataclass
class AdamConfig:
    """optim.hpp:7-12"""
    lr: float = 2e-4
    beta1: float = 0.5
    beta2: float = 0.999
    eps: float = 1e-8


@dataclass
class GroupSpec:
    arch: Arch
    class_ids: list[int]
    batch: int = 64
    epochs: int = 1
    per_label: int = 64
    base_seed: int = 1
    adam: AdamConfig = field(default_factory=AdamConfig)
    clamp: float = 1e-7
    init_std: float = 0.02
    math: int = N.MATH_FP32_SIMT
    threads: int = 8
    device: int = 0


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class LabelGroup:
    """All (G, D) pairs of the given labels on one GPU, stepping in lockstep.

    Each label keeps the reference worker semantics: its own stream
    Rng(derive_seed(base_seed, class_id)) driving the epoch shuffle and the
    latents z1, z2; G/D initialised from derive_seed(worker_seed, 1 / 2).
    """

    def __init__(self, spec: GroupSpec):
        self.spec = spec
        L = N.lib()
        self._ids = (C.c_int * len(spec.class_ids))(*spec.class_ids)
        a = spec.arch
        cfg = N.GroupConfig(
            gen_spec=a.gen.encode(), disc_spec=a.disc.encode(), C=a.image[0], H=a.image[1], W=a.image[2],
            d_z=a.d_z, n_labels=len(spec.class_ids), class_ids=self._ids, base_seed=spec.base_seed,
            batch=spec.batch, epochs=spec.epochs, per_label=spec.per_label, lr=spec.adam.lr,
            beta1=spec.adam.beta1, beta2=spec.adam.beta2, eps=spec.adam.eps, clamp=spec.clamp,
            init_std=spec.init_std, math=spec.math, threads=spec.threads, device=spec.device)
        self._cfg = cfg
        h = C.c_void_p()
        N.check(L.pg_group_create(C.byref(cfg), C.byref(h)), "pg_group_create")
        self._h = h

    # ---- lifecycle ----
    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().pg_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_labels(self) -> int:
        return len(self.spec.class_ids)

    # ---- data ----
    def set_dataset(self, images01: np.ndarray) -> None:
        """images01: [n_labels][per_label][C][H][W] in [0,1] (shard order)."""
        x = np.ascontiguousarray(images01, dtype=np.float32)
        N.check(N.lib().pg_group_set_dataset(self._h, _fptr(x)), "set_dataset")

    def generate_dataset(self, data_seed: int) -> None:
        N.check(N.lib().pg_group_generate_dataset(self._h, data_seed), "generate_dataset")

    # ---- training ----
    def train_steps(self, n: int) -> int:
        """n steps of the worker protocol on the device-resident dataset."""
        return N.check(N.lib().pg_group_train_steps(self._h, n), "train_steps")

    def train_step(self, real01: np.ndarray) -> list[StepReport]:
        """One reference train_step per label on a host batch [n_labels][B][C][H][W]."""
        x = np.ascontiguousarray(real01, dtype=np.float32)
        B = x.shape[1]
        rep = np.zeros((self.n_labels, 4), np.float64)
        N.check(N.lib().pg_group_train_step(self._h, _fptr(x), B, _dptr(rep)), "train_step")
        return [StepReport(*r) for r in rep]

    def train_step_inputs(self, real01: np.ndarray, z1: np.ndarray, z2: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(real01, dtype=np.float32)
        a = np.ascontiguousarray(z1, dtype=np.float32)
        b = np.ascontiguousarray(z2, dtype=np.float32)
        rep = np.zeros((self.n_labels, 4), np.float64)
        N.check(N.lib().pg_group_train_step_inputs(self._h, _fptr(x), _fptr(a), _fptr(b), x.shape[1], _dptr(rep)),
                "train_step_inputs")
        return rep

    def last_device_ms(self) -> float:
        return float(N.lib().pg_group_last_ms(self._h))

    def sync(self) -> None:
        N.check(N.lib().pg_group_sync(self._h), "sync")

    # ---- state (reference layouts, f64) ----
    def get(self, label_index: int, field_code: int) -> np.ndarray:
        L = N.lib()
        n = N.check(L.pg_group_get(self._h, label_index, field_code, None, 0), "get")
        out = np.zeros(n, np.float64)
        N.check(L.pg_group_get(self._h, label_index, field_code, _dptr(out), n), "get")
        return out

    def set(self, label_index: int, field_code: int, values: np.ndarray) -> None:
        v = np.ascontiguousarray(values, dtype=np.float64)
        N.check(N.lib().pg_group_set(self._h, label_index, field_code, _dptr(v), v.size), "set")

    def reports(self, label_index: int) -> np.ndarray:
        return self.get(label_index, N.F_REPORTS).reshape(-1, 4)

    def failed(self) -> np.ndarray:
        f = np.zeros(self.n_labels, np.int32)
        N.check(N.lib().pg_group_failed(self._h, f.ctypes.data_as(C.POINTER(C.c_int))), "failed")
        return f

    def generate(self, n: int, seed: int) -> np.ndarray:
        c, h, w = self.spec.arch.image
        out = np.zeros((self.n_labels, n, c, h, w), np.float32)
        N.check(N.lib().pg_group_generate(self._h, n, seed, _fptr(out)), "generate")
        return out

    def save_checkpoint(self, label: int, path: str) -> None:
        """save_gan_pair (src/checkpoint.cpp:91-139) for label index `label`."""
        N.check(N.lib().pg_group_save_checkpoint(self._h, label, str(path).encode()), "save_checkpoint")

    def load_checkpoint(self, label: int, path: str) -> None:
        """load_gan_pair (src/checkpoint.cpp:141-194) into label index `label`."""
        N.check(N.lib().pg_group_load_checkpoint(self._h, label, str(path).encode()), "load_checkpoint")

    def mixture_sample(self, priors, n: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
        """mixture_sample (partition.cpp:182-227) over this group's labels in
        order: (samples [n][C][H][W] in [0,1], class indices [n])."""
        import ctypes as C
        c, h, w = self.spec.arch.image
        pri = np.ascontiguousarray(priors, np.float64)
        if pri.shape != (self.n_labels,):
            raise ValueError("mixture_sample: prior length does not match pair count")
        out = np.zeros((n, c, h, w), np.float32)
        ids = np.zeros(n, np.int32)
        N.check(N.lib().pg_group_mixture_sample(self._h, pri.ctypes.data_as(C.POINTER(C.c_double)), n, seed,
                                                _fptr(out), ids.ctypes.data_as(C.POINTER(C.c_int))), "mixture_sample")
        return out, ids

    def capture_masks(self, on: bool = True) -> None:
        """Parity instrumentation: record every step's ReLU / LeakyReLU masks
        (pg_group_capture_masks)."""
        N.check(N.lib().pg_group_capture_masks(self._h, 1 if on else 0), "capture_masks")

    def masks(self, label_index: int) -> np.ndarray:
        """the last step's masks of one label, bytes in the oracle MaskTape order"""
        L = N.lib()
        n = N.check(L.pg_group_get_masks(self._h, label_index, None, 0), "get_masks")
        out = np.zeros(n, np.uint8)
        if n:
            N.check(L.pg_group_get_masks(self._h, label_index, out.ctypes.data_as(C.POINTER(C.c_uint8)), n),
                    "get_masks")
        return out

    def sizes(self) -> dict:
        out = (C.c_longlong * 4)()
        N.check(N.lib().pg_group_sizes(self._h, out), "sizes")
        return dict(gen_params=out[0], disc_params=out[1], gen_arena=out[2], disc_arena=out[3])


def make_group(cfg: int, class_ids: list[int], **kw) -> LabelGroup:
    return LabelGroup(GroupSpec(arch=baseline_arch(cfg), class_ids=list(class_ids), **kw))


def derive_seed(base: int, stream: int) -> int:
    return int(N.lib().pg_derive_seed(base, stream))


def shard_begin(n_labels: int, n_gpus: int, g: int) -> int:
    return int(N.lib().pg_shard_begin(n_labels, n_gpus, g))


def cosine_label(shape: tuple[int, int, int], per_label: int, seed: int, label: int) -> np.ndarray:
    c, h, w = shape
    out = np.zeros((per_label, c, h, w), np.float64)
    N.check(N.lib().pg_cosine_label(c, h, w, per_label, seed, label, _dptr(out)), "cosine_label")
    return out


def partition_by_label(labels, k: int) -> list[np.ndarray]:
    """partition.cpp:40-56: stable index list per class; errors on out-of-range
    labels and empty classes."""
    labels = np.asarray(labels)
    if k < 1:
        raise ValueError("partition_by_label: k must be >= 1")
    if labels.size == 0:
        raise ValueError("partition_by_label: empty label vector")
    bad = np.nonzero((labels < 0) | (labels >= k))[0]
    if bad.size:
        i = int(bad[0])
        raise IndexError(f"label {int(labels[i])} at index {i} outside [0, {k})")
    shards = [np.nonzero(labels == j)[0] for j in range(k)]
    for j, s in enumerate(shards):
        if s.size == 0:
            raise ValueError(f"class {j} has no samples")
    return shards


def estimate_priors(shards) -> tuple[np.ndarray, np.ndarray]:
    """partition.cpp:58-74: per-class counts and counts / total, in class
    order; shards are (class_id, indices) pairs covering classes 0..k-1."""
    shards = list(shards)
    if not shards:
        raise ValueError("estimate_priors: no shards")
    counts = np.zeros(len(shards), np.int64)
    for cid, idx in shards:
        if cid < 0 or cid >= len(shards):
            raise ValueError(f"shard class id {cid} out of range")
        if len(idx) == 0:
            raise ValueError(f"class {cid} has no samples")
        counts[cid] = len(idx)
    return counts, counts / counts.sum()
