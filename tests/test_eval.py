"""Evaluation metrics (src/eval.cpp) through the native library, pinned by the
reference's own known-answer and property tests (tests/test_eval.cpp:42-238).
Host arithmetic only: runs without a GPU."""
import numpy as np
import pytest

from paper_2102_10485_b200 import _native as N
from paper_2102_10485_b200.evaluate import anova_f, anova_per_channel, inception_score, softmax_rows


def test_softmax_rows_uniform_onehot_and_formula():  # test_eval.cpp:42-69
    p = softmax_rows(np.full((2, 4), 0.3))
    assert np.allclose(p, 0.25, rtol=1e-12, atol=0)
    big = np.array([[500.0, 0.0, 0.0, 0.0]])
    p = softmax_rows(big)
    assert abs(p[0, 0] - 1.0) < 1e-9 and p[0, 1] < 1e-9
    x = np.random.default_rng(3).normal(size=(5, 4))
    ref = np.exp(x) / np.exp(x).sum(1, keepdims=True)
    assert np.abs(softmax_rows(x) - ref).max() < 1e-12


def test_inception_score_floor_and_ceiling():  # test_eval.cpp:71-84
    floor = inception_score(np.full((40, 5), 0.2), 4)
    assert all(abs(s - 1.0) < 1e-12 for s in floor.split_scores) and floor.stddev == 0.0
    k, n = 10, 100
    onehot = np.zeros((n, k))
    onehot[np.arange(n), np.arange(n) % k] = 1.0
    ceil = inception_score(onehot, 10)
    assert abs(ceil.mean - 10.0) < 1e-9 and all(abs(s - 10.0) < 1e-9 for s in ceil.split_scores)


def test_inception_score_brute_force_example():  # test_eval.cpp:86-100
    rows = np.array([[0.9, 0.1], [0.8, 0.2], [0.5, 0.5]] * 2)
    sr = inception_score(rows, 2)
    assert abs(sr.split_scores[0] - 1.076488453988641) < 1e-12 * 1.08
    assert abs(sr.split_scores[1] - 1.076488453988641) < 1e-12 * 1.08
    assert abs(sr.stddev) < 1e-12


def test_inception_score_bounds_permutation_and_errors():  # test_eval.cpp:102-126
    rng = np.random.default_rng(44)
    for _ in range(100):
        n, k = 10 + int(rng.integers(30)), 2 + int(rng.integers(6))
        p = rng.random((n, k))
        p /= p.sum(1, keepdims=True)
        sr = inception_score(p, 1 + int(rng.integers(5)))
        assert all(1.0 - 1e-12 <= s <= k + 1e-12 for s in sr.split_scores)
    p = rng.random((24, 4))
    p /= p.sum(1, keepdims=True)
    base = inception_score(p, 2)
    perm = [5, 3, 11, 0, 7, 2, 9, 1, 10, 4, 6, 8]
    q = p.copy()
    q[:12] = p[perm]
    assert abs(base.split_scores[0] - inception_score(q, 2).split_scores[0]) < 1e-12
    with pytest.raises(N.PgError, match="cannot fill"):
        inception_score(p, 25)
    with pytest.raises(N.PgError, match="sums to"):
        inception_score(p * 1.5, 2)


def test_anova_f_hand_and_degenerate():  # test_eval.cpp:159-167
    assert abs(anova_f([[0, 2], [1, 3]]) - 0.5) < 1e-12
    assert anova_f([[1.0, 2.0], [1.0, 2.0]]) == 0.0
    assert np.isinf(anova_f([[0.0, 0.0], [1.0, 1.0]]))
    for bad in ([[1.0, 2.0]], [[1.0], []], [[1.0], [2.0]]):
        with pytest.raises(N.PgError):
            anova_f(bad)


def test_anova_brute_force_and_affine_invariance():  # test_eval.cpp:169-207
    rng = np.random.default_rng(9)
    for _ in range(200):
        k = 2 + int(rng.integers(4))
        groups = [list(rng.normal(size=2 + int(rng.integers(6))) + rng.integers(3)) for _ in range(k)]
        allv = np.concatenate(groups)
        grand = allv.mean()
        ssb = sum(len(g) * (np.mean(g) - grand) ** 2 for g in groups)
        ssw = sum(((np.asarray(g) - np.mean(g)) ** 2).sum() for g in groups)
        f_oracle = (ssb / (k - 1)) / (ssw / (len(allv) - k))
        f = anova_f(groups)
        assert abs(f - f_oracle) < 1e-10 * max(1.0, f_oracle)
        mapped = [[-3.7 * v + 11.0 for v in g] for g in groups]
        assert abs(anova_f(mapped) - f) <= 1e-9 * max(1.0, f)


def test_anova_per_channel_constant_classes_is_infinite():  # test_eval.cpp:209-221
    labels = np.array([0, 0, 1, 1, 2, 2, 3, 3])
    images = np.repeat((labels / 4.0)[:, None, None, None], 4, axis=2).reshape(8, 1, 2, 2)
    f = anova_per_channel(images, labels, 4)
    assert f.shape == (1,) and np.isinf(f[0])
    with pytest.raises(N.PgError, match="out of range"):
        anova_per_channel(images, labels + 1, 4)


def test_anova_per_channel_separates_shifted_classes():  # the property of test_eval.cpp:240-
    rng = np.random.default_rng(5)
    labels = np.repeat(np.arange(3), 20)
    images = rng.normal(size=(60, 2, 4, 4)).astype(np.float32)
    images[:, 0] += labels[:, None, None] * 2.0  # channel 0 separates the classes, channel 1 does not
    f = anova_per_channel(images, labels, 3)
    assert f[0] > 100 and f[1] < 10
