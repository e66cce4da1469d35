"""Host-side logic of the product against the oracle, bit for bit: seed
derivation, the cosine-field dataset, label sharding, partition_by_label."""
import numpy as np
import pytest

from paper_2102_10485_b200 import cosine_label, derive_seed, partition_by_label, shard_begin


def test_derive_seed_matches_oracle(native, oracle):
    for base, sid in [(0, 0), (1, 2), (2024, 7), (2**63 + 5, 2**32 - 1), (123, 999)]:
        assert derive_seed(base, sid) == oracle.derive_seed(base, sid)


@pytest.mark.parametrize("shape", [(1, 28, 28), (3, 32, 32), (3, 64, 64)])
def test_cosine_dataset_bit_identical(native, oracle, shape):
    for label in (0, 5, 999):
        a = cosine_label(shape, 3, seed=11, label=label)
        b = oracle.dataset_label(shape, 3, seed=11, label=label)
        assert a.shape == b.shape
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
        assert a.min() >= 0.0 and a.max() <= 1.0


def test_shards_balanced_contiguous_cover(native):
    for n, p in [(10, 8), (100, 8), (1000, 8), (125, 1), (250, 2), (13, 4), (7, 7)]:
        bounds = [shard_begin(n, p, g) for g in range(p + 1)]
        assert bounds[0] == 0 and bounds[-1] == n
        sizes = np.diff(bounds)
        assert sizes.min() >= 0 and sizes.max() - sizes.min() <= 1
    # weak-scaling sweep: 125 labels per GPU at every N
    for gpus in (1, 2, 4, 8):
        sizes = np.diff([shard_begin(125 * gpus, gpus, g) for g in range(gpus + 1)])
        assert (sizes == 125).all()


def test_partition_by_label_matches_oracle(oracle):
    import ctypes as C
    rng = np.random.default_rng(3)
    labels = rng.integers(0, 10, size=5000).astype(np.int32)
    ours = partition_by_label(labels, 10)
    counts = np.zeros(10, np.int64)
    idx = np.zeros(5000, np.int64)
    oracle.check(oracle.lib().or_partition(labels.ctypes.data_as(C.POINTER(C.c_int)), 5000, 10,
                                           counts.ctypes.data_as(C.POINTER(C.c_long)),
                                           idx.ctypes.data_as(C.POINTER(C.c_long))))
    at = 0
    for j in range(10):
        assert np.array_equal(ours[j], idx[at:at + counts[j]])
        at += counts[j]


def test_partition_errors():
    with pytest.raises(IndexError):
        partition_by_label([0, 3], 2)
    with pytest.raises(ValueError, match="class 1 has no samples"):
        partition_by_label([0, 0], 2)
