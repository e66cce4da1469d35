"""Multi-process (world size 2, gloo, CPU) coverage of the label-sharded path:
each rank owns a contiguous label block, runs its labels independently (here:
the CPU oracle stands in for the per-GPU label group, as the checker), and the
final gather reassembles per-label samples and loss statistics on rank 0 in
label order — identical to running all labels in one process."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_10485_b200.distributed import gather_to_root, max_over_ranks, shard_range


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_labels, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle_lib
    labels = list(shard_range(n_labels, world, rank))
    # per-rank label block: one step of the c1 worker protocol per label
    orc = oracle_lib.OracleGroup(64, 1, len(labels), 32, 16, first_label=labels[0], data_seed=3, base_seed=7,
                                 threads=2)
    orc.step(1)
    stats = torch.tensor(np.stack([orc.get(i, 10)[-4:] for i in range(len(labels))]))
    idx = torch.tensor(np.stack([orc.get(i, 11) for i in range(len(labels))]))
    slow = max_over_ranks(float(rank + 1))
    all_stats = gather_to_root(stats, n_labels, world, rank)
    all_idx = gather_to_root(idx, n_labels, world, rank)
    if rank == 0:
        np.savez(out_path, stats=all_stats.numpy(), idx=all_idx.numpy(), slow=slow)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_partition_labels():
    for n, world in [(10, 2), (10, 3), (125 * 2, 2), (7, 4)]:
        got = [list(shard_range(n, world, r)) for r in range(world)]
        assert sum(got, []) == list(range(n))
        sizes = [len(g) for g in got]
        assert max(sizes) - min(sizes) <= 1


@pytest.mark.timeout(300)
def test_two_rank_gloo_shard_and_gather_equals_single_process(tmp_path):
    import oracle_lib
    oracle_lib.build()
    n_labels, world = 5, 2
    out = tmp_path / "gathered.npz"
    mp.start_processes(_worker, args=(world, _free_port(), n_labels, str(out)), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    # same labels in one process
    ref = oracle_lib.OracleGroup(64, 1, n_labels, 32, 16, data_seed=3, base_seed=7, threads=2)
    ref.step(1)
    ref_stats = np.stack([ref.get(i, 10)[-4:] for i in range(n_labels)])
    ref_idx = np.stack([ref.get(i, 11) for i in range(n_labels)])
    # per-label streams are independent of the sharding: bitwise equal
    assert np.array_equal(got["stats"], ref_stats)
    # batch rows are dataset rows of each process's label-blocked dataset:
    # subtract the block offsets to compare shard positions
    first = {i: r.start for r in (shard_range(n_labels, world, k) for k in range(world)) for i in r}
    local = np.array([(i - first[i]) * 32 for i in range(n_labels)])[:, None]
    assert np.array_equal(got["idx"] - local, ref_idx - (np.arange(n_labels)[:, None] * 32))
    assert float(got["slow"]) == world
