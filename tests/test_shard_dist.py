"""The N>1 sweep path on CPU: world_size 2 over gloo.

Covers what bench.py does across ranks, minus the CUDA solve: each rank
builds its own weak-scaling shard of the global instance stream, the shards
concatenate to the single-process stream (shard invariance of the inputs),
per-rank summary statistics (computed here by the C oracle, standing in for
the GPU results) all-reduce to the single-process summary -- the per-instance
decision hashes' sum and XOR bit for bit -- and the job time is the max over
ranks."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import checkers as ck
from paper_2206_06304_b200 import profile_heavy
from paper_2206_06304_b200.shard import (BLOCK, make_instances, max_over_ranks, reduce_summary,
                                         shard_range, summary_stats)

PER_RANK, M = 40, 9


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        prof = profile_heavy(M)
        lo, hi = shard_range(PER_RANK, rank, world)
        users = make_instances(prof, M, lo, hi, seed=3)
        ip, og = ck.oracle_ipssa(prof, users), ck.oracle_og(prof, users)
        stats, hashes = summary_stats(np, ip, og)
        summ = reduce_summary((torch.as_tensor(stats), torch.as_tensor(hashes)), dist)
        slow = max_over_ranks(1.0 + rank, dist)
        out[rank] = (lo, hi, users["deadline"].copy(), summ, slow)
    finally:
        dist.destroy_process_group()


def test_shard_ranges_partition_the_stream():
    assert shard_range(10, 0, 1) == (0, 10)
    assert [shard_range(10, r, 4) for r in range(4)] == [(0, 10), (10, 20), (20, 30), (30, 40)]
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_instances_independent_of_sharding():
    prof = profile_heavy(6)
    whole = make_instances(prof, 6, 0, BLOCK + 100, seed=5)
    a = make_instances(prof, 6, 0, 4000, seed=5)
    b = make_instances(prof, 6, 4000, BLOCK + 100, seed=5)
    for k in whole:
        np.testing.assert_array_equal(whole[k], np.concatenate([a[k], b[k]]))


def test_world2_gloo_sweep_reduction():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True,
                       start_method="fork")
    prof = profile_heavy(M)
    users = make_instances(prof, M, 0, PER_RANK * world, seed=3)
    expect = reduce_summary(summary_stats(np, ck.oracle_ipssa(prof, users),
                                          ck.oracle_og(prof, users)))
    np.testing.assert_array_equal(np.concatenate([out[r][2] for r in range(world)]),
                                  users["deadline"])
    for r in range(world):
        lo, hi, _, summ, slow = out[r]
        assert (lo, hi) == (PER_RANK * r, PER_RANK * (r + 1))
        assert slow == float(world)  # max over ranks
        for k, v in expect.items():
            if k.startswith("decision_hash"):  # decisions: exact, whatever the sharding
                assert summ[k] == v, k
            else:  # energies: a sum of two partial sums vs one sum -> allow rounding
                assert summ[k] == pytest.approx(v, rel=1e-12), k
    assert expect["failed_instances"] == 0
