"""Evaluation of generated samples — the reference's eval.cpp metrics
(softmax_rows, inception_score, anova_f, anova_per_channel; src/eval.cpp:18-211)
through the native library (host C++, f64, same arithmetic and errors)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N


def _d(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass
class ScoreReport:
    """eval.hpp ScoreReport"""
    split_scores: list[float]
    mean: float
    stddev: float
    n_splits: int


def softmax_rows(logits: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(logits, np.float64)
    out = np.empty_like(x)
    N.check(N.lib().pg_softmax_rows(_d(x), x.shape[0], x.size // x.shape[0], _d(out)), "softmax_rows")
    return out


def inception_score(probs: np.ndarray, n_splits: int) -> ScoreReport:
    p = np.ascontiguousarray(probs, np.float64)
    if p.ndim != 2:
        raise ValueError("inception_score: probs must be [N, K]")
    splits = np.zeros(max(n_splits, 1), np.float64)
    mean, std = C.c_double(), C.c_double()
    N.check(N.lib().pg_inception_score(_d(p), p.shape[0], p.shape[1], n_splits, _d(splits), C.byref(mean),
                                       C.byref(std)), "inception_score")
    return ScoreReport(list(splits[:n_splits]), mean.value, std.value, n_splits)


def anova_f(groups: list) -> float:
    sizes = np.asarray([len(g) for g in groups], np.int64)
    vals = np.ascontiguousarray(np.concatenate([np.asarray(g, np.float64) for g in groups]) if len(groups) else
                                np.zeros(0), np.float64)
    f = C.c_double()
    N.check(N.lib().pg_anova_f(_d(vals), sizes.ctypes.data_as(C.POINTER(C.c_long)), len(groups), C.byref(f)),
            "anova_f")
    return f.value


def anova_per_channel(images: np.ndarray, labels: np.ndarray, k: int) -> np.ndarray:
    """images [n][C][H][W], labels [n] in [0, k): F per channel over the per-image spatial means."""
    x = np.ascontiguousarray(images, np.float32)
    lab = np.ascontiguousarray(labels, np.int32)
    n, c, h, w = x.shape
    f = np.zeros(c, np.float64)
    N.check(N.lib().pg_anova_per_channel(x.ctypes.data_as(C.POINTER(C.c_float)), lab.ctypes.data_as(C.POINTER(C.c_int)),
                                         n, c, h, w, k, _d(f)), "anova_per_channel")
    return f
