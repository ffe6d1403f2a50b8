"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 host path:
contiguous stream sharding, max-over-ranks timing, and the gather of
per-stream results, with the CPU oracle standing in for the per-rank compute.
A sharded job must give exactly the single-process result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2106_11594_b200 import sharding, workloads


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle

    b0, b1 = sharding.shard_range(B, world, rank)
    rows, tg = workloads.host_batch("c5", list(range(b0, b1)), n=96)
    o = oracle.ingest(rows, tg, r_cap=16, logs=False)
    ranks = sharding.gather_streams(torch.as_tensor(o["rank"]))
    x = sharding.gather_streams(torch.as_tensor(oracle.solution(o)))
    t = sharding.max_over_ranks(1.0 + rank)
    total = sharding.sum_over_ranks(float(b1 - b0))
    if rank == 0:
        out["ranks"] = ranks.numpy()
        out["x"] = x.numpy()
        out["t"] = t
        out["total"] = total
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_contiguous_and_complete():
    B, world = 64, 4
    got = [sharding.shard_range(B, world, r) for r in range(world)]
    assert got == [(0, 16), (16, 32), (32, 48), (48, 64)]
    with pytest.raises(ValueError):
        sharding.shard_range(10, 4, 0)
    with pytest.raises(ValueError):
        sharding.shard_range(8, 2, 2)


def test_two_rank_gloo_job_equals_single_process():
    from oracle import oracle

    B, world = 8, 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), B, out), nprocs=world, join=True)
    rows, tg = workloads.host_batch("c5", list(range(B)), n=96)
    ref = oracle.ingest(rows, tg, r_cap=16, logs=False)
    assert np.array_equal(out["ranks"], ref["rank"])
    assert np.array_equal(out["x"], oracle.solution(ref))
    assert out["t"] == 2.0 and out["total"] == float(B)


def test_stream_bytes_do_not_depend_on_sharding():
    # host recipe keyed by global index: shard-local generation == global slice
    a, ya = workloads.host_batch("c5", [5, 6], n=32)
    b, yb = workloads.host_batch("c5", list(range(8)), n=32)
    assert np.array_equal(a, b[5:7]) and np.array_equal(ya, yb[5:7])
